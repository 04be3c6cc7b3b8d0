"""Debug: one 2D D2H copy of 49152 rows vs 12 copies of 4096 rows (per-copy overhead)."""
import time
import torch
from cuda.bindings import runtime as rt
rows, pitch, S = 49152, 4008, 5
w = pitch // S
dev = torch.empty(rows * pitch, dtype=torch.uint8, device="cuda")
host = torch.empty(rows * pitch, dtype=torch.uint8, pin_memory=True)
st = torch.cuda.Stream()
for parts in (1, 12, 48):
    per = rows // parts
    def go():
        for s in range(S):
            for k in range(parts):
                r0 = k * per
                rt.cudaMemcpy2DAsync(host.data_ptr() + r0 * pitch + s * w, pitch, dev.data_ptr() + r0 * pitch + s * w,
                                     pitch, w, per, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost, st.cuda_stream)
        st.synchronize()
    go()
    t0 = time.perf_counter(); go(); go(); dt = (time.perf_counter() - t0) / 2
    t1 = time.perf_counter()
    for s in range(S):
        for k in range(parts):
            r0 = k * per
            rt.cudaMemcpy2DAsync(host.data_ptr() + r0 * pitch + s * w, pitch, dev.data_ptr() + r0 * pitch + s * w,
                                 pitch, w, per, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost, st.cuda_stream)
    enq = time.perf_counter() - t1
    st.synchronize()
    print(f"{parts:3d} copies x {per} rows per segment: {rows * pitch / dt / 1e9:.1f} GB/s, enqueue {enq*1e3:.2f} ms for {S*parts} copies")
