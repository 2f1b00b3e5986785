import torch, time
n = 3613007872 // 4
h = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
s = torch.cuda.Stream()
for chunk in (n, n // 32):
    for _ in range(2):
        torch.cuda.synchronize(); t = time.perf_counter()
        with torch.cuda.stream(s):
            for o in range(0, n, chunk):
                d[o:o + chunk].copy_(h[o:o + chunk], non_blocking=True)
        s.synchronize(); dt = time.perf_counter() - t
    print(f"chunk {chunk*4/1e6:.0f} MB: {n*4/dt/1e9:.1f} GB/s ({dt*1e3:.1f} ms)")
# two streams alternating chunks
s2 = torch.cuda.Stream(); chunk = n // 32
torch.cuda.synchronize(); t = time.perf_counter()
for i, o in enumerate(range(0, n, chunk)):
    with torch.cuda.stream(s if i % 2 == 0 else s2):
        d[o:o + chunk].copy_(h[o:o + chunk], non_blocking=True)
torch.cuda.synchronize(); dt = time.perf_counter() - t
print(f"2 streams, {chunk*4/1e6:.0f} MB chunks: {n*4/dt/1e9:.1f} GB/s")
