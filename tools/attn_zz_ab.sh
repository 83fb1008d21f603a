# Attention item order: zig-zag rounds (in-tree) vs plain striding (xv/nozz.so).
timeout 300 python -m pytest tests/test_mla_attn_gpu.py tests/test_mla.py -q -x -m gpu 2>&1 | tail -1
for r in 1 2; do
  for L in 8192 32768; do
    echo "zz:   $(timeout 120 python tools/time_attn.py $L 16 2>&1 | head -1)"
    echo "nozz: $(BD_LIB_PATH=xv/nozz.so timeout 120 python tools/time_attn.py $L 16 2>&1 | head -1)"
  done
done
