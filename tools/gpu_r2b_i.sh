mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_stage_spec.py tests/test_gpu_parity.py tests/test_gpu_init.py tests/test_gpu_airpf.py tests/test_gpu_adaptive.py tests/test_gpu_fullsize.py tests/test_gpu_filter.py -x -q > gpurun_out/i_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/i_pytest.log
B="timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e"
$B > gpurun_out/i_C4.json 2>&1
$B --config C3 > gpurun_out/i_C3.json 2>&1
$B --airpf 1 > gpurun_out/i_C4_airpf1.json 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_pass1 -s 3 -c 1 -o gpurun_out/i_pass1 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/i_ncu1.log 2>&1
