cat > /tmp/one.py <<'PY'
import torch, paper_2510_01718_b200 as bd
dev="cuda:0"; L,d,d_h,n=8192,512,128,16; K,N=d-d_h,n*d_h
x=torch.randn(L,d,device=dev); ck=torch.randn(K,N,device=dev)/8; cv=torch.randn(K,N,device=dev)/8
for _ in range(3): bd.fused_kv_proj_grouped(x,[(ck,d_h,n,bd.Tag.FIRST),(cv,d_h,n,bd.Tag.LAST)],check_finite=False)
torch.cuda.synchronize()
PY
PYTHONPATH=$PWD ncu --set full --clock-control none --import-source on -k regex:kv_proj_exact -s 2 -c 1 -o gpurun_out/exact64 python /tmp/one.py > gpurun_out/ncu_exact.log 2>&1
tail -3 gpurun_out/ncu_exact.log
