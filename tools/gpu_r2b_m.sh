mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_airpf.py tests/test_gpu_airpf2.py tests/test_gpu_fullsize.py tests/test_gpu_multinomial.py tests/test_gpu_relabel.py tests/test_gpu_sharded.py -x -q > gpurun_out/m_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/m_pytest.log
B="timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e"
for M in 128 512 2048 8192; do $B --config C5 --M $M > gpurun_out/m_C5_M$M.json 2>&1; $B --config C5 --M $M --airpf 1 > gpurun_out/m_C5_M${M}_airpf.json 2>&1; done
$B --config C2 > gpurun_out/m_C2.json 2>&1
$B --config C2 --airpf 1 > gpurun_out/m_C2_airpf.json 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_pass1 -s 2 -c 1 -o gpurun_out/m_pass1_c5 python bench.py --config C5 --M 8192 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/m_ncu_c5.log 2>&1
