# interleaved attention timing: the in-tree build vs abtmp/base.so (the previous kernel,
# built in the container and shipped for the A/B)
timeout 300 python -m pytest tests/test_mla_attn_gpu.py -m gpu -x -q --timeout 300 > gpurun_out/attn_tests.log 2>&1
echo "attn tests rc=$?"; tail -1 gpurun_out/attn_tests.log
for r in 1 2 3; do
  echo -n "new:  "; timeout 120 python tools/time_attn.py 32768 16 2>&1 | head -1
  echo -n "base: "; BD_LIB_PATH=abtmp/base.so timeout 120 python tools/time_attn.py 32768 16 2>&1 | head -1
done
