"""Raw PCIe probe: D2H/H2D bandwidth of pinned copies of various sizes, alone and while a
compute kernel runs (the overlap case of the segmented rollout)."""
import time, torch
N = 560 << 20
d = torch.empty(N, dtype=torch.uint8, device="cuda")
h = torch.empty(N, dtype=torch.uint8, pin_memory=True)
s = torch.cuda.Stream()
for chunk in [N, N // 8, N // 64, N // 512]:
    torch.cuda.synchronize()
    for rep in range(2):
        t0 = time.perf_counter()
        with torch.cuda.stream(s):
            for o in range(0, N, chunk):
                h[o:o + chunk].copy_(d[o:o + chunk], non_blocking=True)
        s.synchronize()
        dt = time.perf_counter() - t0
    print(f"D2H chunk {chunk >> 20} MiB: {N / dt / 1e9:.1f} GB/s", flush=True)
t0 = time.perf_counter(); d.copy_(h, non_blocking=True); torch.cuda.synchronize(); print(f"H2D: {N / (time.perf_counter() - t0) / 1e9:.1f} GB/s")
# concurrent with a long compute kernel on the default stream
a = torch.randn(8192, 8192, device="cuda")
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20): a = a @ a * 1e-4
with torch.cuda.stream(s):
    h.copy_(d, non_blocking=True)
s.synchronize(); t1 = time.perf_counter(); torch.cuda.synchronize()
print(f"D2H while GEMMs run: {N / (t1 - t0) / 1e9:.1f} GB/s (lower bound)")
