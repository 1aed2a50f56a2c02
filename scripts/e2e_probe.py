"""Probe of the host-buffer path on the GPU box: raw pinned copy rates on the
state-sized float64 buffers, and RingStepper.step_host over chunk counts, with
and without the D2H of the new cells. One JSON line."""

import json
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2303_08058_b200 import _native as N  # noqa: E402
from paper_2303_08058_b200.ring import RingStepper  # noqa: E402


def gpu_ms(fn, reps=5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def main():
    S = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
    N.init(0)
    st = RingStepper(S, max_steps=512)
    host = torch.empty((S, 512), dtype=torch.float64, pin_memory=True)
    host2 = torch.empty((S, 512), dtype=torch.float64, pin_memory=True)
    host.copy_(st.cells)
    stats = torch.empty(2, dtype=torch.float64, pin_memory=True)
    d = torch.empty_like(st.cells)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    out = {"subgrids": S, "bytes": S * 4096}
    out["h2d_ms"] = gpu_ms(lambda: d.copy_(host, non_blocking=True))
    out["d2h_ms"] = gpu_ms(lambda: host2.copy_(d, non_blocking=True))

    def both():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            d.copy_(host, non_blocking=True)
        with torch.cuda.stream(s2):
            host2.copy_(st.cells, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    out["h2d_and_d2h_concurrent_ms"] = gpu_ms(both)
    for chunks in (1, 2, 4, 8, 16, 32):
        out[f"step_host_c{chunks}_ms"] = gpu_ms(lambda: st.step_host(host, host, stats, chunks))
        out[f"step_host_noD2H_c{chunks}_ms"] = gpu_ms(
            lambda: st.step_host(host, None, stats, chunks))
    t0 = time.perf_counter()
    for _ in range(10):
        st.step_host(host, host, stats, 16)
    out["enqueue_ms_c16"] = (time.perf_counter() - t0) * 100
    torch.cuda.synchronize()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
