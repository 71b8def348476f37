mkdir -p gpurun_out
B="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e"
for r in 1 2; do
PF_PASS1_PERSIST=0 timeout 300 $B > gpurun_out/b_C4_p0_$r.json 2>&1
PF_PASS1_PERSIST=1 timeout 300 $B > gpurun_out/b_C4_p1_$r.json 2>&1
done
timeout 1200 python -m pytest tests/test_gpu_stage_spec.py tests/test_gpu_parity.py -x -q > gpurun_out/b_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/b_pytest.log
