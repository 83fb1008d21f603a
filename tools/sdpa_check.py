import torch, time, torch.nn.functional as F
from torch.nn.attention import sdpa_kernel, SDPBackend
L,H,D=32768,16,192
q=torch.randn(1,H,L,D,device='cuda',dtype=torch.float16)
k=torch.randn(1,H,L,D,device='cuda',dtype=torch.float16)
v=torch.randn(1,H,L,D,device='cuda',dtype=torch.float16)
v128=torch.randn(1,H,L,128,device='cuda',dtype=torch.float16)
def t(fn):
    fn(); torch.cuda.synchronize()
    s=time.time()
    for _ in range(3): fn()
    torch.cuda.synchronize(); return (time.time()-s)/3*1e3
for name,b in [("flash",SDPBackend.FLASH_ATTENTION),("eff",SDPBackend.EFFICIENT_ATTENTION),("cudnn",SDPBackend.CUDNN_ATTENTION)]:
    for vv,lab in [(v,"v192"),(v128,"v128")]:
        try:
            with sdpa_kernel([b]):
                ms=t(lambda: F.scaled_dot_product_attention(q,k,vv,is_causal=True,scale=D**-0.5))
            print(name,lab,f"{ms:.2f} ms")
        except Exception as e:
            print(name,lab,"ERR",str(e)[:100])
ms=t(lambda: F.scaled_dot_product_attention(q,k,v,is_causal=True,scale=D**-0.5)); print("default 4d v192", ms)
q3=q[0];k3=k[0];v3=v[0]
ms=t(lambda: F.scaled_dot_product_attention(q3,k3,v3,is_causal=True,scale=D**-0.5)); print("default 3d", ms)
