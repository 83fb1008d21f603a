# persistent kernel tile width A/B: parity under both widths, then graph-timed short launches
mkdir -p gpurun_out
timeout ${TT:-400} python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/tile_tests.log 2>&1
echo "tests (default widths) rc=$?"; tail -2 gpurun_out/tile_tests.log
BD_TILE_N=256 timeout 300 python -m pytest tests/test_kv_proj_gpu.py -m gpu -x -q --timeout 300 > gpurun_out/tile_tests256.log 2>&1
echo "tests (BD_TILE_N=256) rc=$?"; tail -2 gpurun_out/tile_tests256.log
BD_TILE_N=128 timeout 300 python -m pytest tests/test_kv_proj_gpu.py -m gpu -x -q --timeout 300 -k "not cfg2_full and not fullsize" > gpurun_out/tile_tests128.log 2>&1
echo "tests (BD_TILE_N=128) rc=$?"; tail -2 gpurun_out/tile_tests128.log
for v in "X=1" "BD_TILE_N=256" "BD_SMALL_MAXL=128" "BD_SMALL_MAXL=128 BD_TILE_N=256"; do
  echo "== $v"; env $v NDT=1 timeout 120 python tools/decode_ab.py ${LS:-256 512 1024}
done
