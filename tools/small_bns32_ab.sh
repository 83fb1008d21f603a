# Small-L kernel: 32-column blocks (64-byte swizzle B panel; auto when every CTA gets its
# own SM) vs the 64-column blocks (BD_SMALL_BNS=64); parity first.
timeout 600 python -m pytest tests/test_kv_proj_gpu.py -q -x -m gpu 2>&1 | tail -2
for r in 1 2; do
  echo "auto:  $(timeout 300 python tools/time_short.py)"
  echo "bns64: $(BD_SMALL_BNS=64 timeout 300 python tools/time_short.py)"
done
