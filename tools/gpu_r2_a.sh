# round 2, call A: new parity tests first, then the whole GPU suite, then one bench line
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_init.py tests/test_gpu_sharded.py tests/test_gpu_parity.py tests/test_gpu_airpf.py -x -q > gpurun_out/r2a_new.log 2>&1; echo "rc=$?" >> gpurun_out/r2a_new.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2a_all.log 2>&1; echo "rc=$?" >> gpurun_out/r2a_all.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err; echo "rc=$?" >> gpurun_out/r2a_bench.err
