mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:k_stages -c 2 -o gpurun_out/k_stages_rot python bench.py --theta 0.5 --rotate --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/k_ncu_rot.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_pass1 -s 2 -c 1 -o gpurun_out/k_pass1_c5 python bench.py --config C5 --M 8192 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/k_ncu_c5.log 2>&1
