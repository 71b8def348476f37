mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/c_launches.csv $CMD > gpurun_out/c_ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_pass1 -s 3 -c 1 -o gpurun_out/c_pass1 $CMD > gpurun_out/c_ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_stages -s 9 -c 1 -o gpurun_out/c_stages $CMD > gpurun_out/c_ncu2.log 2>&1
