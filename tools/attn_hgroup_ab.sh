# Attention work-item order A/B: heads per scheduling group (BD_ATTN_HGROUP; 16 = every
# head in flight, the previous order).  Parity tests first.
timeout 600 python -m pytest tests/test_mla_attn_gpu.py tests/test_mla.py -q -x -m gpu 2>&1 | tail -2
for r in 1 2; do
  for gsz in 16 1 2 3 4 8; do
    echo "hgroup $gsz: $(BD_ATTN_HGROUP=$gsz timeout 300 python tools/time_attn.py 32768 16 2>&1 | head -1)"
  done
done
echo "default: $(timeout 300 python tools/time_attn.py 32768 16 2>&1 | head -3)"
