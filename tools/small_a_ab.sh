C=paper_2510_01718_b200/csrc
python tools/knobs_small_a.py > /dev/null
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -shared -I$C -DUNSHARED_A \
  -o /tmp/ua.so $C/capi.cu $C/kv_proj_exact.cu xb/kv_proj_tc_ua.cu $C/mla_attn.cu
for r in 1 2; do
  echo "== shared A (shipped)"; timeout 120 python tools/small_a_ab.py
  echo "== unshared A";        BD_LIB_PATH=/tmp/ua.so timeout 120 python tools/small_a_ab.py
done
