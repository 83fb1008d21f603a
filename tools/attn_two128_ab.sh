# The parked 128-key two-query-tile kernel (tools/experiments/mla_attn_2tile.cu) with the
# shipped item order (head groups + zig-zag rounds), built as xv/two128.so, vs in-tree.
BD_LIB_PATH=xv/two128.so timeout 300 python -m pytest tests/test_mla_attn_gpu.py -q -x -m gpu 2>&1 | tail -1
for r in 1 2; do
  for L in 8192 32768; do
    echo "in-tree: $(timeout 120 python tools/time_attn.py $L 16 2>&1 | head -1)"
    echo "two128:  $(BD_LIB_PATH=xv/two128.so timeout 120 python tools/time_attn.py $L 16 2>&1 | head -1)"
  done
done
