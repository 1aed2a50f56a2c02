"""Where K6's per-launch fixed cost goes (config 2): per-CTA globaltimer
stamps of a TB_HYDRO_VARIANT=1020 launch (= 508 + stamps) after an L2
flush — launch head (entry spread, first staging wait), steady rounds, tail
(exit spread) — beside the 508 launch's event time."""
import ctypes
import json
import os
import sys

os.environ.setdefault("TB_HYDRO_VARIANT", "1020")
import torch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_08058_b200 import _native as N  # noqa: E402
from paper_2303_08058_b200 import hydro  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
dev = torch.device("cuda", 0)
I, dx = hydro.rotating_star(S, device=dev)
U = hydro.with_ghosts(I)
du = torch.empty((S, 5, 8, 8, 8), dtype=torch.float64, device=dev)
am = torch.empty(S, dtype=torch.float64, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for _ in range(3):
    hydro.hydro_flux(U, dx, out=du, amax=am)
rows = []
for rep in range(5):
    flush.fill_(1)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    hydro.hydro_flux(U, dx, out=du, amax=am)
    b.record()
    torch.cuda.synchronize()
    n = 296
    buf = (ctypes.c_ulonglong * (4 * n))()
    N.call("tb_hydro_stamps", buf, n)
    st = [[buf[4 * i + j] for j in range(4)] for i in range(n)]
    t0 = min(r[0] for r in st)
    us = lambda x: round((x - t0) / 1e3, 2)  # noqa: E731
    ent = sorted(us(r[0]) for r in st)
    first = sorted(us(r[1]) for r in st)
    lastf = sorted(us(r[2]) for r in st)
    ex = sorted(us(r[3]) for r in st)
    rows.append({"event_ms": round(a.elapsed_time(b), 4),
                 "entry_us": [ent[0], ent[len(ent) // 2], ent[-1]],
                 "first_staged_us": [first[0], first[len(first) // 2], first[-1]],
                 "last_faces_us": [lastf[0], lastf[len(lastf) // 2], lastf[-1]],
                 "exit_us": [ex[0], ex[len(ex) // 2], ex[-1]]})
for r in rows:
    print(json.dumps(r))
