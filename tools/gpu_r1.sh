#!/bin/bash
# Round-1 GPU pass: parity tests, smoke, bench, ncu launch list, ncu full capture of the top kernel.
set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 50 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
CMD2="python tools/run_steps.py C4 268435456 64 3"
timeout 600 $CMD2 > gpurun_out/plain2.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_pass1 -s 1 -c 1 -o gpurun_out/prof_pass1 $CMD2 > gpurun_out/ncu_full.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_compose -s 2 -c 1 -o gpurun_out/prof_compose $CMD2 > gpurun_out/ncu_full2.log 2>&1
ls -la gpurun_out
