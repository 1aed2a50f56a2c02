"""Timeline of chained RingStepper.step_host calls: when each chunk's H2D,
K2 and D2H completed (timing events on each stream), relative to the first
step's start. Prints one JSON line per step plus the steady-state period."""

import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2303_08058_b200 import _native as N  # noqa: E402
from paper_2303_08058_b200 import ring as R  # noqa: E402


def main():
    S = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
    chunks = int(sys.argv[2]) if len(sys.argv) > 2 else 16
    N.init(0)
    st = R.RingStepper(S, max_steps=64)
    host = torch.empty((S, 512), dtype=torch.float64, pin_memory=True)
    host.copy_(st.cells)
    stats = torch.empty(2, dtype=torch.float64, pin_memory=True)
    for _ in range(3):
        st.step_host(host, host, stats, chunks)
    torch.cuda.synchronize()
    # instrument: wrap Event so every event the step records is a timing event
    made = []
    orig = torch.cuda.Event

    def timing_event(*a, **k):
        e = orig(enable_timing=True)
        made.append(e)
        return e

    R.torch.cuda.Event = timing_event
    t0 = orig(enable_timing=True)
    t0.record()
    steps = 4
    per_step = []
    for _ in range(steps):
        n0 = len(made)
        st.step_host(host, host, stats, chunks, join=False)
        per_step.append(made[n0:])
    st.join_host()
    t1 = orig(enable_timing=True)
    t1.record()
    torch.cuda.synchronize()
    R.torch.cuda.Event = orig
    total = t0.elapsed_time(t1)
    for k, evs in enumerate(per_step):
        # order of creation in step_host: h2d[c], k2[c], d2h[c], faces, done
        c = chunks
        h2d, k2, d2h = evs[0:c], evs[c:2 * c], evs[2 * c:3 * c]
        rel = lambda e: round(t0.elapsed_time(e), 3)  # noqa: E731
        print(json.dumps({"step": k, "h2d_done": [rel(e) for e in h2d],
                          "k2_done": [rel(e) for e in k2],
                          "d2h_done": [rel(e) for e in d2h]}))
    print(json.dumps({"total_ms": total, "per_step_ms": total / steps}))


if __name__ == "__main__":
    main()
