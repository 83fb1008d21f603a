# mirror-schedule A/B: parity (default; forced on where legal; forced off), then the
# head-sharded per-rank workload (tools/shard_sim.py) with the schedule off and on
mkdir -p gpurun_out
timeout 400 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/swap_tests.log 2>&1
echo "tests rc=$?"; tail -1 gpurun_out/swap_tests.log
BD_SWAP=1 timeout 300 python -m pytest tests/test_kv_proj_gpu.py tests/test_fullsize_gpu.py -m gpu -x -q --timeout 300 -k "not cfg5" > gpurun_out/swap_tests1.log 2>&1
echo "tests (BD_SWAP=1) rc=$?"; tail -1 gpurun_out/swap_tests1.log
BD_SWAP=0 timeout 300 python -m pytest tests/test_kv_proj_gpu.py -m gpu -x -q --timeout 300 -k mirror > gpurun_out/swap_tests0.log 2>&1
echo "tests (BD_SWAP=0) rc=$?"; tail -1 gpurun_out/swap_tests0.log
for v in 0 -1 1; do echo "== BD_SWAP=$v"; BD_SWAP=$v timeout 200 python tools/shard_sim.py; done
