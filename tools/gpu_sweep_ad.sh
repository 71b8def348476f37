mkdir -p gpurun_out
bash tools/sweep2.sh > gpurun_out/sweep_ad.txt 2>&1
for th in 0.5 0.9; do timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --theta $th 2>&1 | tail -1 > gpurun_out/bench_ad_$th.json; done
