mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_airpf2.py tests/test_gpu_airpf.py tests/test_gpu_parity.py tests/test_gpu_adaptive.py tests/test_gpu_sharded.py tests/test_gpu_fullsize.py -x -q > gpurun_out/k_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/k_pytest.log
TAG=k VARIANTS_FILE=tools/sweep_r2_k.txt bash tools/sweep_env.sh
