# Small-L kernel for 128 < L <= 512: single CTAs per 128-row block (default) vs CTA pairs
# (BD_SMALL_PAIRS=1); also wide problems on the small kernel (BD_SMALL_WIDE=1).
timeout 600 python -m pytest tests/test_kv_proj_gpu.py tests/test_callers_gpu.py -q -x -m gpu 2>&1 | tail -1
for r in 1 2; do
  echo "single: $(timeout 300 python tools/time_short.py)"
  echo "pairs:  $(BD_SMALL_PAIRS=1 timeout 300 python tools/time_short.py)"
  echo "wide:   $(BD_SMALL_WIDE=1 timeout 300 python tools/time_short.py)"
done
