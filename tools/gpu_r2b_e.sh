mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_stage_spec.py -x -q > gpurun_out/e_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/e_pytest.log
PF_WSC_VARIANT=1 timeout 600 python -m pytest tests/test_gpu_stage_spec.py -x -q > gpurun_out/e_pytest_v1.log 2>&1; echo "rc=$?" >> gpurun_out/e_pytest_v1.log
B="timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e"
$B > gpurun_out/e_C4_v0.json 2>&1
for v in 1 2 3; do PF_WSC_VARIANT=$v $B > gpurun_out/e_C4_wsc$v.json 2>&1; done
for h in 20000 2000 200; do PF_WS_SLEEP_NS=$h $B > gpurun_out/e_C4_v0_h$h.json 2>&1; PF_WSC_VARIANT=1 PF_WS_SLEEP_NS=$h $B > gpurun_out/e_C4_wsc1_h$h.json 2>&1; done
$B > gpurun_out/e_C4_v0b.json 2>&1
