"""Timeline probe of RingStepper.step_host (host-buffer path) on the GPU box.

Prints per-step GPU time, host enqueue time, and — for one instrumented step
— when each chunk's H2D / K2 / D2H finished relative to the step start.
"""

import json
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2303_08058_b200 import _native as N  # noqa: E402
from paper_2303_08058_b200.ring import RingStepper, chunk_bounds  # noqa: E402


def main():
    S = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
    chunks = int(sys.argv[2]) if len(sys.argv) > 2 else 16
    N.init(0)
    st = RingStepper(S, max_steps=64)
    host = torch.empty((S, 512), dtype=torch.float64, pin_memory=True)
    host.copy_(st.cells)
    stats = torch.empty(2, dtype=torch.float64, pin_memory=True)
    torch.cuda.synchronize()
    out = {"subgrids": S, "chunks": chunks, "steps": []}
    for k in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        t0 = time.perf_counter()
        st.step_host(host, host, stats, chunks=chunks)
        t_enq = time.perf_counter() - t0
        e1.record()
        torch.cuda.synchronize()
        out["steps"].append({"gpu_ms": e0.elapsed_time(e1), "enqueue_ms": t_enq * 1e3})
    # plain serial path for comparison: one H2D, one step, one D2H
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    st.cells.copy_(host, non_blocking=True)
    st.step()
    host.copy_(st.cells, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    out["serial_ms"] = e0.elapsed_time(e1)
    # raw copies of the same size for reference
    d = torch.empty_like(st.cells)
    for name, fn in [("h2d_only", lambda: d.copy_(host, non_blocking=True)),
                     ("d2h_only", lambda: host.copy_(d, non_blocking=True))]:
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        out[name + "_ms"] = e0.elapsed_time(e1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
