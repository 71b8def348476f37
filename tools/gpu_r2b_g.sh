mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/g_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g_pytest.log
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/g_launches.csv $CMD > gpurun_out/g_ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_pass1 -s 3 -c 1 -o gpurun_out/g_pass1 $CMD > gpurun_out/g_ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_stages -s 9 -c 1 -o gpurun_out/g_stages $CMD > gpurun_out/g_ncu2.log 2>&1
timeout 900 python bench.py > gpurun_out/g_bench_C4.json 2> gpurun_out/g_bench_C4.err
timeout 600 python bench.py --impl reference > gpurun_out/g_bench_ref.json 2> gpurun_out/g_bench_ref.err
for c in C1 C2 C3; do timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/g_bench_$c.json 2>&1; done
timeout 300 python bench.py --config C5 --M 8192 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/g_bench_C5_8192.json 2>&1
timeout 300 python bench.py --airpf 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/g_bench_C4_airpf1.json 2>&1
timeout 300 python bench.py --airpf 1 --theta 0.5 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/g_bench_C4_airpf2.json 2>&1
timeout 300 python bench.py --theta 0.5 --rotate --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/g_bench_C4_theta05_rot.json 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/g_smoke.log 2>&1
