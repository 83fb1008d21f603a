# Attention producer: K and V requested independently (in-tree) vs in lock-step
# (xv/lockstep.so); parity first.
timeout 300 python -m pytest tests/test_mla_attn_gpu.py -q -x -m gpu 2>&1 | tail -1
for r in 1 2; do
  for L in 8192 32768; do
    echo "decoupled: $(timeout 120 python tools/time_attn.py $L 16 2>&1 | head -1)"
    echo "lockstep:  $(BD_LIB_PATH=xv/lockstep.so timeout 120 python tools/time_attn.py $L 16 2>&1 | head -1)"
  done
done
