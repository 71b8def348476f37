mkdir -p gpurun_out
PF_PLAN_VERBOSE=1 timeout 120 python bench.py --config C5 --M 8 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bb_plan.txt 2>&1
TAG=bb VARIANTS_FILE=tools/sweep_r2_bb.txt bash tools/sweep_env.sh
