mkdir -p gpurun_out
./tools/micro/draw_bench > gpurun_out/d_draw.txt 2>&1
TAG=d bash tools/gpu_iter_r2.sh
PF_PASS1_SHFL=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/d_bench_shfl.json 2>&1
