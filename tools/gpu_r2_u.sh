mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_graph.py tests/test_gpu_filter.py tests/test_gpu_parity.py tests/test_gpu_sharded.py tests/test_gpu_adaptive.py -x -q > gpurun_out/u_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/u_pytest.log
