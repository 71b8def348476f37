mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stage_spec.py -x -q > gpurun_out/c_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/c_pytest.log
for pf in 0 1 2 3; do PF_STAGE_PREFETCH=$pf timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c_bench_C4_pf$pf.json 2>&1; done
PF_PASS1_SPEC=0 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c_bench_C4_nop1spec.json 2>&1
for w in 12 20; do PF_STAGE_WS_WALK32=$w timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c_bench_C4_w$w.json 2>&1; done
timeout 300 python bench.py --config C3 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/c_bench_C3.json 2>&1
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
ncu --set full --clock-control none --import-source on -k regex:k_pass1 -s 3 -c 1 -o gpurun_out/c_pass1 $CMD > gpurun_out/c_ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_stages -s 9 -c 1 -o gpurun_out/c_stages $CMD > gpurun_out/c_ncu2.log 2>&1
