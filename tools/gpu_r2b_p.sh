mkdir -p gpurun_out
B="timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e"
for M in 2 4 8 32; do PF_PLAN_VERBOSE=1 $B --config C5 --M $M > gpurun_out/p_C5_M$M.json 2> gpurun_out/p_C5_M$M.err; done
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/p_launches_c5m2.csv python bench.py --config C5 --M 2 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/p_launches_c5m8.csv python bench.py --config C5 --M 8 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
