# round 2 perf iteration: parity subset, then a C4 bench line (per-kernel CUDA-event times)
# usage: TAG=x TESTS="tests/test_gpu_parity.py ..." bash tools/gpu_iter_r2.sh
mkdir -p gpurun_out
T=${TAG:-it}
timeout 900 python -m pytest ${TESTS:-tests/test_gpu_parity.py tests/test_gpu_airpf.py tests/test_gpu_adaptive.py} -x -q > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "rc=$?" >> gpurun_out/${T}_bench.err
