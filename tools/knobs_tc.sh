# timing-only bisection of the persistent kernel's cfg2 tile period (tools/knobs_tc.py)

C=paper_2510_01718_b200/csrc
mkdir -p exp gpurun_out
python tools/instrument.py > /dev/null
python tools/knobs_tc.py > /dev/null
for k in NONE NOMMA NOSTG NOSTORE; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -I$C \
    -D$k -o exp/k_$k.so $C/capi.cu $C/kv_proj_exact.cu exp/kv_proj_tc_tl.cu $C/mla_attn.cu &
done
wait
for k in NONE NOMMA NOSTG NOSTORE; do
  echo "== $k"
  BD_LIB_PATH=exp/k_$k.so timeout 120 python tools/sweep_l.py $k 8192
  BD_LIB_PATH=exp/k_$k.so timeout 120 python tools/timeline.py 8192 20 | grep -E "period|b_full|mma window|epi start|epi end|7-tile"
done
