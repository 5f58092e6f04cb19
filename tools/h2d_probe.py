import torch,time
x=torch.empty(2**31//4*4, dtype=torch.uint8, pin_memory=True); d=torch.empty_like(x, device='cuda')
for _ in range(2): d.copy_(x, non_blocking=True)
torch.cuda.synchronize(); t=time.perf_counter()
for _ in range(5): d.copy_(x, non_blocking=True)
torch.cuda.synchronize(); print("H2D GB/s", 5*x.numel()/(time.perf_counter()-t)/1e9)
