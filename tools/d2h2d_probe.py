"""Debug: D2H throughput of 2D (strided host rows) copies vs row width."""
import time
import torch
from cuda.bindings import runtime as rt
rows = 49152
st = torch.cuda.Stream()
for total_w in (8016, 4008, 2000, 1000):       # host row pitch (bytes per episode)
    for S in (4, 8):
        w = total_w // S
        dev = torch.empty(rows * w, dtype=torch.uint8, device="cuda")
        host = torch.empty(rows * total_w, dtype=torch.uint8, pin_memory=True)
        def go():
            for s in range(S):
                rt.cudaMemcpy2DAsync(host.data_ptr() + s * w, total_w, dev.data_ptr(), w, w, rows,
                                     rt.cudaMemcpyKind.cudaMemcpyDeviceToHost, st.cuda_stream)
            st.synchronize()
        go()
        t0 = time.perf_counter(); go(); go(); dt = (time.perf_counter() - t0) / 2
        print(f"pitch {total_w:5d} width {w:5d}: {S * rows * w / dt / 1e9:6.1f} GB/s")
dev = torch.empty(400 << 20, dtype=torch.uint8, device="cuda"); host = torch.empty(400 << 20, dtype=torch.uint8, pin_memory=True)
host.copy_(dev); torch.cuda.synchronize()
t0 = time.perf_counter(); host.copy_(dev); torch.cuda.synchronize(); print(f"1D: {400*2**20/(time.perf_counter()-t0)/1e9:.1f} GB/s")
