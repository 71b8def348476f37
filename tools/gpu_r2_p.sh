mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/p_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/p_pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/p_bench_C4.json 2> gpurun_out/p_bench_C4.err
timeout 300 python bench.py --config C1 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/p_bench_C1.json 2>&1
timeout 300 python bench.py --airpf 1 --theta 0.5 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/p_bench_C4_airpf2.json 2>&1
timeout 600 python tools/loopback_bench.py C4 8 peer 3 > gpurun_out/p_loop_peer.txt 2>&1
timeout 600 python tools/loopback_bench.py C4 8 relabel 3 > gpurun_out/p_loop_relabel.txt 2>&1
