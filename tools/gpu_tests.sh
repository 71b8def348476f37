# GPU test pass: one file first (-x, verbose tail), then the whole GPU suite.
mkdir -p gpurun_out
timeout 900 python -m pytest ${FIRST:-tests/test_gpu_airpf.py} -x -q > gpurun_out/pytest_first.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_first.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_all.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_all.log
