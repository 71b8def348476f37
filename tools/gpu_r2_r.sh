mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_overlap.py -x -q > gpurun_out/r_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r_pytest.log
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/r_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r_launches.csv $CMD > gpurun_out/r_ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_pass1 -s 3 -c 1 -o gpurun_out/r_pass1 $CMD > gpurun_out/r_ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_stages -s 9 -c 1 -o gpurun_out/r_stages $CMD > gpurun_out/r_ncu2.log 2>&1
