for v in "BD_DECODE_KPS=6" "BD_DECODE=0"; do
  for a in "cfg2 64" "paper 64"; do env $v timeout 60 python tools/prof_decode.py $a; done
done
BD_DECODE_KPS=6 timeout 300 ncu --set full -k regex:decode -s 5 -c 1 -o gpurun_out/dec_full python tools/prof_decode.py cfg2 64 > gpurun_out/dec_ncu.log 2>&1
BD_DECODE=0 timeout 300 ncu --set full -k regex:small -s 5 -c 1 -o gpurun_out/small_full python tools/prof_decode.py cfg2 64 >> gpurun_out/dec_ncu.log 2>&1
tail -3 gpurun_out/dec_ncu.log
