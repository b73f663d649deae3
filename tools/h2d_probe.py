import torch, time
x = torch.empty(31_405_288, dtype=torch.uint8).pin_memory()
y = torch.empty_like(x, device='cuda')
for _ in range(3): y.copy_(x, non_blocking=True)
torch.cuda.synchronize()
for n in (1, 4, 8):
    chunk = x.numel() // n
    t = time.perf_counter()
    for r in range(20):
        for k in range(n):
            y[k*chunk:(k+1)*chunk].copy_(x[k*chunk:(k+1)*chunk], non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 20
    print(f"H2D 31.4MB in {n} chunks: {dt*1e3:.3f} ms  {31.4/dt/1e3:.1f} GB/s")
x2 = torch.empty(31_405_288, dtype=torch.uint8)  # pageable
t = time.perf_counter()
for r in range(5): y.copy_(x2)
torch.cuda.synchronize(); dt=(time.perf_counter()-t)/5
print(f"pageable H2D: {dt*1e3:.3f} ms {31.4/dt/1e3:.1f} GB/s")
