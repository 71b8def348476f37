mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_stage_spec.py tests/test_gpu_adaptive.py tests/test_gpu_airpf2.py -x -q > gpurun_out/q_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/q_pytest.log
B="timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e"
$B --theta 0.5 > gpurun_out/q_C4_theta05.json 2>&1
$B --theta 0.5 --rotate > gpurun_out/q_C4_theta05_rot.json 2>&1
$B --theta 0.9 > gpurun_out/q_C4_theta09.json 2>&1
$B --theta 0.9 --rotate > gpurun_out/q_C4_theta09_rot.json 2>&1
$B --airpf 1 --theta 0.5 > gpurun_out/q_C4_airpf2.json 2>&1
