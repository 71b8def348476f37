mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_adaptive.py -x -q > gpurun_out/pytest_adaptive.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_adaptive.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_all.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_all.log
