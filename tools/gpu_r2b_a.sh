mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/a_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/a_pytest.log
timeout 600 python bench.py > gpurun_out/a_bench_C4.json 2> gpurun_out/a_bench_C4.err
timeout 300 python bench.py --config C1 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/a_bench_C1.json 2>&1
timeout 300 python bench.py --config C5 --M 8192 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/a_bench_C5_8192.json 2>&1
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/a_launches.csv $CMD > gpurun_out/a_ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_pass1 -s 3 -c 1 -o gpurun_out/a_pass1 $CMD > gpurun_out/a_ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_stages -s 9 -c 1 -o gpurun_out/a_stages $CMD > gpurun_out/a_ncu2.log 2>&1
