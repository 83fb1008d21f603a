# Interleaved A/B of xv/*.so library builds with tools/time_short.py (ROUNDS rounds).
for r in $(seq ${ROUNDS:-3}); do
  for v in xv/*.so; do echo "$v: $(BD_LIB_PATH=$v timeout 300 python tools/time_short.py)"; done
done
