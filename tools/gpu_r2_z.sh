mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_adaptive.py tests/test_gpu_sharded.py tests/test_gpu_airpf.py tests/test_gpu_poison.py tests/test_gpu_filter.py -x -q > gpurun_out/z_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/z_pytest.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/z_bench.json 2>&1
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --config C2 > gpurun_out/z_bench_C2.json 2>&1
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --config C3 > gpurun_out/z_bench_C3.json 2>&1
