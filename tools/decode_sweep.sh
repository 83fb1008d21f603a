# decode-kernel A/B on one box: parity tests, then the graph-timed sweep for several
# k-block splits / column blocks against the older small-L kernel (BD_DECODE=0)
mkdir -p gpurun_out
timeout ${TT:-240} python -m pytest tests/test_kv_proj_gpu.py -m gpu -x -q --timeout 300 \
  -k "${TESTK:-decode or small_l or fuzz or strided or launch_counter}" > gpurun_out/decode_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/decode_tests.log
for v in ${VARIANTS:-kps1 kps2 kps3 kps6 old}; do
  case $v in
    old) env="BD_DECODE=0" ;;
    kps*) env="BD_DECODE_KPS=${v#kps}" ;;
    bns*) env="BD_DECODE_BNS=${v#bns}" ;;
    *) env="$v" ;;
  esac
  echo "== $v ($env)"
  env $env NDT=${NDT:-1} timeout ${AT:-90} python tools/decode_ab.py ${LS:-1 64 128}
done
