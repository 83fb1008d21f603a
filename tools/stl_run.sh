# stamped small-L kernel: timelines (default) or the timing-only knob bisection (KNOBS=1)
set -e
C=paper_2510_01718_b200/csrc
python tools/instrument_small.py
build() { nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -I$C "$@" $C/capi.cu $C/kv_proj_exact.cu xb/kv_proj_tc_stl.cu $C/mla_attn.cu; }
if [ -n "$KNOBS" ]; then
  KL=${KLIST:-NONE SKIP_LOADS SKIP_MMA SKIP_STORES SKIP_REP ALL}
  for k in $KL; do
    f=$(echo $k | sed 's/ALL/SKIP_LOADS+SKIP_MMA+SKIP_STORES+SKIP_REP/; s/^/-D/; s/+/ -D/g')
    build $f -o /tmp/k_$k.so &
  done
  wait
  for k in $KL; do
    for a in ${CASES:-cfg2:64}; do
      echo "== knob $k"; RING=${RING:-warm} BD_LIB_PATH=/tmp/k_$k.so timeout 120 python tools/small_timeline2.py ${a/:/ } | ${FILTER:-head -1}
    done
  done
  exit 0
fi
build -o /tmp/stl.so
for r in ${RINGS:-cold}; do
for a in ${CASES:-cfg2:1 cfg2:64 paper:64}; do
  RING=$r BD_LIB_PATH=/tmp/stl.so timeout 120 python tools/small_timeline2.py ${a/:/ }
done
done
