C=paper_2510_01718_b200/csrc
mkdir -p exp
python tools/instrument.py > /dev/null
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -I$C \
  -o exp/tl.so $C/capi.cu $C/kv_proj_exact.cu exp/kv_proj_tc_tl.cu $C/mla_attn.cu
for a in "256 20 128 single" "512 20 128 single" "8192 20"; do
  echo "== $a"; BD_LIB_PATH=exp/tl.so timeout 120 python tools/timeline.py $a
done
