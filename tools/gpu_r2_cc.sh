mkdir -p gpurun_out
for M in 4 8 16 32 128; do PF_PLAN_VERBOSE=1 timeout 120 python bench.py --config C5 --M $M --steps 1 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep "pf plan" > gpurun_out/cc_plan_M$M.txt; done
PF_PLAN_VERBOSE=1 timeout 120 python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep "pf plan" > gpurun_out/cc_plan_C4.txt
PF_PLAN_VERBOSE=1 timeout 120 python bench.py --config C3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep "pf plan" > gpurun_out/cc_plan_C3.txt
TAG=cc VARIANTS_FILE=tools/sweep_r2_cc.txt bash tools/sweep_env.sh
