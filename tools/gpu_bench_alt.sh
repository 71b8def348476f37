# Benchmarks of the NEXT rows (AIRPF, fully adapted) beside the plain step, C4.
mkdir -p gpurun_out
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_plain.json 2> gpurun_out/bench_plain.err
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --airpf 1 > gpurun_out/bench_airpf1.json 2> gpurun_out/bench_airpf1.err
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --airpf 2 > gpurun_out/bench_airpf2.json 2> gpurun_out/bench_airpf2.err
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --airpf 1 --config C3 > gpurun_out/bench_airpf1_C3.json 2>&1
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --airpf 1"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_airpf.csv $CMD > gpurun_out/ncu_airpf.log 2>&1
