mkdir -p gpurun_out
./tools/micro/draw_bench > gpurun_out/f_draw.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_relabel.py tests/test_gpu_sharded.py tests/test_gpu_parity.py -x -q > gpurun_out/f_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/f_pytest.log
