"""Debug: 2D D2H copies (strided host rows) on 1..4 concurrent streams."""
import time
import torch
from cuda.bindings import runtime as rt
rows = 49152
for pitch, S in ((4008, 5), (2000, 5), (1000, 5)):
    w = pitch // S
    dev = torch.empty(rows * pitch, dtype=torch.uint8, device="cuda")
    host = torch.empty(rows * pitch, dtype=torch.uint8, pin_memory=True)
    for ns in (1, 2, 4):
        sts = [torch.cuda.Stream() for _ in range(ns)]
        def go():
            for s in range(S):
                # split the rows of each segment copy across the streams
                per = (rows + ns - 1) // ns
                for k, st in enumerate(sts):
                    r0, r1 = k * per, min(rows, (k + 1) * per)
                    rt.cudaMemcpy2DAsync(host.data_ptr() + r0 * pitch + s * w, pitch, dev.data_ptr() + r0 * pitch + s * w,
                                         pitch, w, r1 - r0, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost, st.cuda_stream)
            for st in sts: st.synchronize()
        go()
        t0 = time.perf_counter(); go(); go(); dt = (time.perf_counter() - t0) / 2
        print(f"pitch {pitch} width {w} streams {ns}: {rows * pitch / dt / 1e9:.1f} GB/s")
