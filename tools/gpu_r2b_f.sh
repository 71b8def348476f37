mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_stage_spec.py -x -q > gpurun_out/f_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/f_pytest.log
B="timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e"
$B > gpurun_out/f_C4_def.json 2>&1
PF_PASS1_MINB=5 $B > gpurun_out/f_C4_minb5.json 2>&1
PF_PASS1_MINB=7 $B > gpurun_out/f_C4_minb7.json 2>&1
PF_PASS1_THREADS=256 PF_PASS1_MINB=3 $B > gpurun_out/f_C4_q1m3.json 2>&1
PF_PASS1_THREADS=256 PF_PASS1_MINB=4 $B > gpurun_out/f_C4_q1m4.json 2>&1
$B > gpurun_out/f_C4_def2.json 2>&1
