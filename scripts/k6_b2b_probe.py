"""K6 at config 2 (4096 sub-grids, inputs 283 MB > the 126 MB L2): launches
back to back (the K2 headline's method) vs after a flushing write vs after a
flushing read; under ncu (--cache-control none) the back-to-back launches'
DRAM bytes show whether any input is re-read from L2."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_08058_b200 import hydro  # noqa: E402

S = 4096
dev = torch.device("cuda", 0)
I, dx = hydro.rotating_star(S, device=dev)
U = hydro.with_ghosts(I)
du = torch.empty((S, 5, 8, 8, 8), dtype=torch.float64, device=dev)
am = torch.empty(S, dtype=torch.float64, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
sink = torch.empty(1, dtype=torch.int64, device=dev)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
for _ in range(3):
    hydro.hydro_flux(U, dx, out=du, amax=am)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(n):
    hydro.hydro_flux(U, dx, out=du, amax=am)
b.record()
torch.cuda.synchronize()
res = {"back_to_back_ms": a.elapsed_time(b) / n}


def timed(prep, reps=n):
    tot = 0.0
    for _ in range(reps):
        prep()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        hydro.hydro_flux(U, dx, out=du, amax=am)
        e1.record()
        torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    return tot / reps


res["flush_write_ms"] = timed(lambda: flush.fill_(1))
res["flush_read_ms"] = timed(lambda: torch.sum(flush.view(torch.int64), dim=0, out=sink.view(())))
print(json.dumps({k: round(v, 4) for k, v in res.items()}))
