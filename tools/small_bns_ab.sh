# small-L single-CTA kernel: the column-block heuristic vs a forced 64 / 128 (BD_SMALL_BNS)
timeout 200 python -m pytest tests/test_kv_proj_gpu.py -m gpu -x -q --timeout 200 -k "small_l or fuzz" > gpurun_out/bns_tests.log 2>&1
echo "tests rc=$?"; tail -1 gpurun_out/bns_tests.log
BD_SMALL_BNS=128 timeout 200 python -m pytest tests/test_kv_proj_gpu.py -m gpu -x -q --timeout 200 -k "small_l or fuzz" > gpurun_out/bns_tests128.log 2>&1
echo "tests (128) rc=$?"; tail -1 gpurun_out/bns_tests128.log
for r in 1 2; do
  for v in 0 64 128; do echo "== BD_SMALL_BNS=$v"; BD_SMALL_BNS=$v NDT=1 timeout 120 python tools/decode_ab.py 1 64 128; done
done
