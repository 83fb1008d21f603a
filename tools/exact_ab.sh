# A/B of exact-kernel (kv_proj_exact.cu) variants on one box: parity tests, then timing of
# the in-tree build and of xv/ variants (tools/time_exact.py).  EXACT_AB_TILES="128 64"
# adds forced-tile runs of the in-tree build.
set -x
timeout 900 python -m pytest tests/test_kv_proj_gpu.py tests/test_callers_gpu.py tests/test_fullsize_gpu.py -x -q -m gpu 2>&1 | tail -4
for r in 1 2; do
echo "== in-tree auto"; timeout 300 python tools/time_exact.py
for t in $EXACT_AB_TILES; do echo "== in-tree tile $t"; BD_EXACT_TILE=$t timeout 300 python tools/time_exact.py; done
for v in xv/*.so; do echo "== $v"; BD_LIB_PATH=$v timeout 300 python tools/time_exact.py; done
done
