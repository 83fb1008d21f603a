# attention kernel A/B: parity, then cfg5-size timing of the in-tree build and of variants
# given as name:flags (built by tools/build_variant.sh into xb/)
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_mla_attn_gpu.py -m gpu -x -q --timeout 300 > gpurun_out/attn_tests.log 2>&1
echo "attn tests rc=$?"; tail -2 gpurun_out/attn_tests.log
for v in ${ATTN_VARIANTS:-}; do
  name=${v%%:*}; flags=${v#*:}
  bash tools/build_variant.sh $name $flags > /dev/null 2>&1 || echo "build $name failed"
done
for r in 1 2 3; do
  echo -n "in-tree: "; timeout 300 python tools/time_attn.py ${ATTN_L:-32768} 16 2>&1 | head -1
  for v in ${ATTN_VARIANTS:-}; do
    name=${v%%:*}
    echo -n "$name: "; BD_LIB_PATH=xb/$name.so timeout 300 python tools/time_attn.py ${ATTN_L:-32768} 16 2>&1 | head -1
  done
done
