# Two-query-tile attention kernel (default) vs the one-tile kernel (BD_ATTN_KERNEL=1):
# parity tests under a timeout, then interleaved timing at 8k and cfg5 (32k) size.
timeout 300 python -m pytest tests/test_mla_attn_gpu.py -q -x -m gpu 2>&1 | tail -3
echo "tests rc=${PIPESTATUS[0]}"
BD_ATTN_KERNEL=1 timeout 300 python -m pytest tests/test_mla_attn_gpu.py -q -x -m gpu 2>&1 | tail -1
for r in 1 2; do
  for L in 8192 32768; do
    echo "k2: $(timeout 120 python tools/time_attn.py $L 16 2>&1 | head -1)"
    echo "k1: $(BD_ATTN_KERNEL=1 timeout 120 python tools/time_attn.py $L 16 2>&1 | head -1)"
  done
done
