"""Where K6's ~16 us per-launch fixed cost comes from (K6): the
same launch timed (a) after a 256 MiB flushing WRITE (bench.py's method),
(b) after a 256 MiB flushing READ (no dirty lines to write back), (c) back to
back without a flush, 20 launches between two events."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import hydro_oracle as h  # noqa: E402  (synthetic inputs only)
from paper_2303_08058_b200.hydro import hydro_flux  # noqa: E402


def main():
    res = {}
    for s in [int(x) for x in (sys.argv[1:] or ["4096", "32768"])]:
        I, dx = h.rotating_star(s)
        U = torch.from_numpy(h.with_ghosts(I)).cuda()
        out = torch.empty((s, 5, 8, 8, 8), dtype=torch.float64, device="cuda")
        amax = torch.empty(s, dtype=torch.float64, device="cuda")
        flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
        sink = torch.empty(1, dtype=torch.int64, device="cuda")
        for _ in range(3):
            hydro_flux(U, dx, out=out, amax=amax)

        def timed(prep, n=20):
            tot = 0.0
            for _ in range(n):
                prep()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                hydro_flux(U, dx, out=out, amax=amax)
                b.record()
                torch.cuda.synchronize()
                tot += a.elapsed_time(b)
            return tot / n

        r = {"flush_write": timed(lambda: flush.fill_(1)),
             "flush_read": timed(lambda: torch.sum(flush.view(torch.int64), dim=0, out=sink)),
             "no_flush_synced": timed(lambda: None)}
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        for _ in range(20):
            hydro_flux(U, dx, out=out, amax=amax)
        b.record()
        torch.cuda.synchronize()
        r["back_to_back"] = a.elapsed_time(b) / 20
        res[s] = {k: round(v, 4) for k, v in r.items()}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
