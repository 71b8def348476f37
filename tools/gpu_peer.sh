# Peer-memory exchange: IPC test, loopback parity, loopback projection (pull vs peer).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_peer_ipc.py tests/test_gpu_sharded.py -x -q > gpurun_out/pytest_peer.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_peer.log
for m in pull peer; do timeout 600 python tools/loopback_bench.py C4 8 $m 5 > gpurun_out/loopback_$m.txt 2>&1; done
