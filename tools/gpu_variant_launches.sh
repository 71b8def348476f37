# ncu launch lists of the next-row variants on C4 (each command first runs clean without ncu)
mkdir -p gpurun_out
for v in "--airpf 1" "--theta 0.5" "--theta 0.5 --rotate" "--multinomial"; do
  tag=$(echo $v | tr -d ' -' | tr '.' 'p')
  CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline $v"
  timeout 600 $CMD > gpurun_out/plain_$tag.log 2>&1 && \
    timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_$tag.csv $CMD > gpurun_out/ncu_$tag.log 2>&1
done
ls gpurun_out/launches_*.csv
