mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_airpf.py tests/test_gpu_airpf2.py tests/test_gpu_adaptive.py tests/test_gpu_fullsize.py -x -q > gpurun_out/w_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/w_pytest.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/w_bench.json 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --config C3 > gpurun_out/w_bench_C3.json 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --config C5 --M 8192 > gpurun_out/w_bench_C5_8192.json 2>&1
