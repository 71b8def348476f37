#!/bin/bash
# GPU evidence pass: parity tests, smoke, bench (ours + reference arm), ncu launch list,
# ncu full captures of k_pass1 and k_stages.  Usage: tools/gpu_evidence.sh <tag>
TAG=${1:-v}
set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
if [ -z "$SKIP_TESTS" ]; then
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
fi
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/plain_$TAG.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1
CMD2="python tools/run_steps.py C4 268435456 64 3"
timeout 600 $CMD2 > gpurun_out/plain2_$TAG.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_pass1 -s 1 -c 1 -o gpurun_out/prof_pass1_$TAG $CMD2 > gpurun_out/ncu_full_pass1_$TAG.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_stages -s 3 -c 1 -o gpurun_out/prof_stages_$TAG $CMD2 > gpurun_out/ncu_full_stages_$TAG.log 2>&1
ls -la gpurun_out
