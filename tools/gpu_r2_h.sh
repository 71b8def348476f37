mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_adaptive.py tests/test_gpu_sharded.py -x -q > gpurun_out/h_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/h_pytest.log
TAG=h VARIANTS_FILE=tools/sweep_r2_h.txt bash tools/sweep_env.sh
