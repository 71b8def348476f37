mkdir -p gpurun_out
./tools/micro/draw_bench > gpurun_out/g_draw.txt 2>&1
TAG=g VARIANTS_FILE=tools/sweep_r2_g.txt bash tools/sweep_env.sh
