mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_adaptive.py tests/test_gpu_sharded.py tests/test_gpu_poison.py -x -q > gpurun_out/x_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/x_pytest.log
TAG=x VARIANTS_FILE=tools/sweep_r2_x.txt bash tools/sweep_env.sh
