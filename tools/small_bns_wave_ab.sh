# Small-L kernel one-wave column blocks (96 at 3 row blocks, 160 at 5): parity, then the
# cfg2 shape at L = 300..640 against the previous choices (BD_SMALL_BNS=128; L > 512 on
# the persistent kernel via BD_SMALL_MAXL=512).
timeout 600 python -m pytest tests/test_kv_proj_gpu.py -q -x -m gpu 2>&1 | tail -1
export TIME_SHORT_CASES="cfg2:300,cfg2:384,cfg2:512,cfg2:600,cfg2:640,cfg2:768"
for r in 1 2; do
  echo "auto:    $(timeout 300 python tools/time_short.py)"
  echo "bns128:  $(BD_SMALL_BNS=128 timeout 300 python tools/time_short.py)"
  echo "maxl512: $(BD_SMALL_MAXL=512 timeout 300 python tools/time_short.py)"
done
