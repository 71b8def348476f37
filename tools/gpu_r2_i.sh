mkdir -p gpurun_out
TAG=i VARIANTS_FILE=tools/sweep_r2_i.txt bash tools/sweep_env.sh
timeout 900 python -m pytest tests/test_gpu_airpf2.py tests/test_gpu_airpf.py tests/test_gpu_parity.py tests/test_gpu_adaptive.py tests/test_gpu_sharded.py -x -q > gpurun_out/i_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/i_pytest.log
