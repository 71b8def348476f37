mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stage_spec.py tests/test_gpu_parity.py tests/test_gpu_init.py tests/test_gpu_airpf.py -x -q > gpurun_out/d_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/d_pytest.log
B="timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e"
$B > gpurun_out/d_C4_v0.json 2>&1
PF_PASS1_VARIANT=1 $B > gpurun_out/d_C4_p1v1.json 2>&1
for v in 1 2 3; do PF_WSC_VARIANT=$v $B > gpurun_out/d_C4_wsc$v.json 2>&1; done
for w in 12 20; do for v in 0 2; do PF_WSC_VARIANT=$v PF_STAGE_WS_WALK32=$w $B > gpurun_out/d_C4_wsc${v}_w$w.json 2>&1; done; done
$B > gpurun_out/d_C4_v0b.json 2>&1
