mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_graph.py tests/test_gpu_filter.py tests/test_gpu_parity.py tests/test_gpu_sharded.py tests/test_gpu_adaptive.py -x -q > gpurun_out/v_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/v_pytest.log
for v in yhost ydev yhost2 ydev2; do
  extra=""; case $v in ydev*) extra="--y-dev";; esac
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e $extra > gpurun_out/v_$v.json 2>&1
done
