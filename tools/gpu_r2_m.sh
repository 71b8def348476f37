mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/m_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_pass1 -s 3 -c 1 -o gpurun_out/m_pass1 $CMD > gpurun_out/m_ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_stages -s 9 -c 1 -o gpurun_out/m_stages $CMD > gpurun_out/m_ncu2.log 2>&1
cat > /tmp/v.txt <<'V'
w12a PF_STAGE_WS_WALK32=12
w10a PF_STAGE_WS_WALK32=10
w16a PF_STAGE_WS_WALK32=16
nows PF_STAGE_WS=0
w12b PF_STAGE_WS_WALK32=12
w10b PF_STAGE_WS_WALK32=10
V
TAG=m VARIANTS_FILE=/tmp/v.txt bash tools/sweep_env.sh
