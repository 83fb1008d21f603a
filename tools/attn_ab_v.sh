# interleaved attention timing: in-tree build vs abtmp/v.so (a variant built in the
# container), plus the variant's attention parity tests
BD_LIB_PATH=abtmp/v.so timeout 300 python -m pytest tests/test_mla_attn_gpu.py -m gpu -x -q --timeout 300 > gpurun_out/attn_v_tests.log 2>&1
echo "variant attn tests rc=$?"; tail -1 gpurun_out/attn_v_tests.log
for r in 1 2 3; do
  echo -n "in-tree: "; timeout 120 python tools/time_attn.py 32768 16 2>&1 | head -1
  echo -n "variant: "; BD_LIB_PATH=abtmp/v.so timeout 120 python tools/time_attn.py 32768 16 2>&1 | head -1
done
