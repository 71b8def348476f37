mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_relabel.py tests/test_gpu_airpf_sharded.py tests/test_gpu_graph.py -x -q > gpurun_out/aa_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/aa_pytest.log
timeout 600 python tools/loopback_bench.py C4 8 relabel 3 > gpurun_out/aa_loop_relabel.txt 2>&1
timeout 600 python tools/loopback_bench.py C4 8 peer 3 > gpurun_out/aa_loop_peer.txt 2>&1
timeout 1200 python tools/c5_sweep.py 4 > gpurun_out/aa_c5_sweep.json 2> gpurun_out/aa_c5_sweep.err
