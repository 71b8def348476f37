mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_overlap.py tests/test_gpu_parity.py tests/test_gpu_adaptive.py tests/test_gpu_sharded.py tests/test_gpu_relabel.py tests/test_gpu_airpf2.py -x -q > gpurun_out/n_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/n_pytest.log
cat > /tmp/v.txt <<'V'
w12 PF_STAGE_WS_WALK32=12
w8 PF_STAGE_WS_WALK32=8
w16 PF_STAGE_WS_WALK32=16
nows PF_STAGE_WS=0
w12b PF_STAGE_WS_WALK32=12
V
TAG=n VARIANTS_FILE=/tmp/v.txt bash tools/sweep_env.sh
