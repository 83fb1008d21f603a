import sys, time
sys.path.insert(0, '.')
import torch, paper_2510_01718_b200 as bd
dev = torch.device('cuda')
L, d, d_h, n = 8192, 512, 128, 16
ck = (torch.randn(384, 2048, device=dev)/8).half(); cv = (torch.randn(384, 2048, device=dev)/8).half()
xh = [torch.randn(L, d).half().pin_memory() for _ in range(2)]
kh = [torch.empty(L, 2048).half().pin_memory() for _ in range(2)]
vh = [torch.empty(L, 2048).half().pin_memory() for _ in range(2)]
specs = [(ck, d_h, n, bd.Tag.FIRST), (cv, d_h, n, bd.Tag.LAST)]
for chunks in (1, 2, 4, 8):
    for i in range(3): bd.fused_kv_proj_grouped_host(xh[i%2], specs, outs=[kh[i%2], vh[i%2]], chunks=chunks)
    torch.cuda.synchronize(); t = time.perf_counter()
    for i in range(30): bd.fused_kv_proj_grouped_host(xh[i%2], specs, outs=[kh[i%2], vh[i%2]], chunks=chunks)
    torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 30
    print(f"chunks {chunks}: {dt*1e3:.3f} ms/step  {L/dt/1e6:.2f} M tok/s")
ref = bd.fused_kv_proj_grouped(xh[0].to(dev), specs)
out = bd.fused_kv_proj_grouped_host(xh[0], specs, chunks=4)
print("equal:", torch.equal(out[0].to(dev), ref[0]), torch.equal(out[1].to(dev), ref[1]))
# raw copy-engine ceiling on this box: one 67 MB D2H and one 8 MB H2D, pinned
src = torch.empty(L, 4096, dtype=torch.half, device=dev)
dst = torch.empty(L, 4096, dtype=torch.half).pin_memory()
for _ in range(3): dst.copy_(src, non_blocking=True)
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(20): dst.copy_(src, non_blocking=True)
torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 20
print(f"D2H {src.numel()*2/1e6:.0f} MB: {dt*1e3:.3f} ms  {src.numel()*2/dt/1e9:.1f} GB/s")
