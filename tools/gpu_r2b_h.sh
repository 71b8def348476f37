mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stage_spec.py -x -q > gpurun_out/h_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/h_pytest.log
B="timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e"
$B > gpurun_out/h_C4_s1.json 2>&1
PF_STAGE_SPEC=3 $B > gpurun_out/h_C4_s3.json 2>&1
for w in 8 12 20 24; do PF_STAGE_SPEC=3 PF_STAGE_WS_WALK32=$w $B > gpurun_out/h_C4_s3_w$w.json 2>&1; done
PF_STAGE_SPEC=3 timeout 300 python bench.py --config C3 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/h_C3_s3.json 2>&1
timeout 300 python bench.py --config C3 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/h_C3_s1.json 2>&1
PF_STAGE_SPEC=3 timeout 300 python bench.py --config C2 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/h_C2_s3.json 2>&1
timeout 300 python bench.py --config C2 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/h_C2_s1.json 2>&1
PF_STAGE_SPEC=3 ncu --set full --clock-control none --import-source on -k regex:k_stages -s 9 -c 1 -o gpurun_out/h_stages3 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/h_ncu.log 2>&1
