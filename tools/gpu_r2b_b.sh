mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stage_spec.py tests/test_gpu_fullsize.py -x -q > gpurun_out/b_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/b_pytest.log
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/b_bench_C4.json 2>&1
PF_STAGE_SPEC=0 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_bench_C4_nospec.json 2>&1
for w in 12 14 18 20; do PF_STAGE_WS_WALK32=$w timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_bench_C4_w$w.json 2>&1; done
timeout 300 python bench.py --config C3 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/b_bench_C3.json 2>&1
timeout 300 python bench.py --config C2 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/b_bench_C2.json 2>&1
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
ncu --set full --clock-control none --import-source on -k regex:k_stages -s 9 -c 1 -o gpurun_out/b_stages $CMD > gpurun_out/b_ncu2.log 2>&1
