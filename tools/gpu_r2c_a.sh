mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/a_smi.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/a_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/a_bench_C4.json 2> gpurun_out/a_bench_C4.err
timeout 600 python bench.py --impl reference > gpurun_out/a_bench_ref.json 2> gpurun_out/a_bench_ref.err
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/a_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/a_pytest.log
