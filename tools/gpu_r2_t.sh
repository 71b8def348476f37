mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_graph.py tests/test_gpu_parity.py tests/test_gpu_sharded.py tests/test_gpu_adaptive.py -x -q > gpurun_out/t_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/t_pytest.log
timeout 300 python bench.py --config C1 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/t_bench_C1.json 2>&1
timeout 300 python bench.py --config C1 --steps 50 --warmup 5 --no-cpu-baseline --graph 0 > gpurun_out/t_bench_C1_nograph.json 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/t_bench_C4.json 2>&1
timeout 300 python bench.py --config C5 --M 8192 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/t_bench_C5_8192.json 2>&1
