mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_stage_spec.py tests/test_gpu_airpf.py tests/test_gpu_airpf2.py tests/test_gpu_airpf_sharded.py -x -q > gpurun_out/o_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/o_pytest.log
B="timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e"
$B --airpf 1 > gpurun_out/o_C4_airpf1.json 2>&1
$B --airpf 2 > gpurun_out/o_C4_airpf2alg6.json 2>&1
$B --airpf 1 --theta 0.5 > gpurun_out/o_C4_airpf2.json 2>&1
PF_PASS1_SPEC=0 $B --airpf 1 > gpurun_out/o_C4_airpf1_nospec.json 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_pass1 -s 2 -c 1 -o gpurun_out/o_pass1_airpf python bench.py --airpf 1 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/o_ncu_airpf.log 2>&1
