mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_stage_spec.py tests/test_gpu_sharded.py tests/test_gpu_overlap.py tests/test_gpu_peer_ipc.py tests/test_gpu_relabel.py -x -q > gpurun_out/s_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s_pytest.log
timeout 900 python tools/loopback_bench.py C4 8 peer 3 > gpurun_out/s_loop_peer8.txt 2>&1
timeout 900 python tools/loopback_bench.py C4 2 peer 3 > gpurun_out/s_loop_peer2.txt 2>&1
timeout 900 python tools/loopback_bench.py C4 4 peer 3 > gpurun_out/s_loop_peer4.txt 2>&1
