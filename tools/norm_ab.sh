# Fused-RMSNorm projection: per-quadrant exchange barriers (in-tree) vs the CTA-wide ones
# (xv/norm_old.so); parity first.
timeout 600 python -m pytest tests/test_kv_proj_gpu.py tests/test_mla.py -q -x -m gpu -k "rmsnorm or norm or mla" 2>&1 | tail -1
for r in 1 2 3; do
  echo "quad: $(timeout 120 python tools/time_rmsnorm.py 2>&1 | tr '\n' ' ')"
  echo "old:  $(BD_LIB_PATH=xv/norm_old.so timeout 120 python tools/time_rmsnorm.py 2>&1 | tr '\n' ' ')"
done
