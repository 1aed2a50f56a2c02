"""K2 A/B helper: µs/step of back-to-back single-device steps at C4 for
20-, 64- and 640-step windows after a 250 ms warm-up. Variants are chosen by
environment (e.g. TB_STEP_ALUMIN=0/1), one process per variant; run
alternately to cancel box drift."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_08058_b200 import _native as N  # noqa: E402
from paper_2303_08058_b200.ring import RingStepper  # noqa: E402

N.init(0)
dev = torch.device("cuda", 0)
subgrids = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
st = RingStepper(subgrids, device=dev, max_steps=200000)


def timed(steps):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        st.step()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / steps


t0 = time.perf_counter()
while time.perf_counter() - t0 < 0.25:
    for _ in range(32):
        st.step()
    torch.cuda.synchronize()
env = {k: v for k, v in os.environ.items() if k.startswith("TB_")}
res = {"env": env, "subgrids": subgrids}
res.update({str(k): [round(timed(k), 2) for _ in range(5)] for k in (20, 64, 640)})
print(json.dumps(res))
