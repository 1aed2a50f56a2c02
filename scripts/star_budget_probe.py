"""Calibration probe for tests/test_gpu_star.py::test_star_conservation_budgets:
per step, the whole-lattice residuals of mass, momentum (vs the gravity
impulse) and energy (vs the gravity work), relative to their scales."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_08058_b200.star import RotatingStarStep  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 4
st = RotatingStarStep(L, device=torch.device("cuda", 0), record_stages=True)


def tot(x):
    return x.sum(dim=(-3, -2, -1))


for k in range(3):
    U0 = st.U.clone()
    st.step()
    torch.cuda.synchronize()
    dt = st.dt.item()
    d = tot(st.U) - tot(U0)
    scale = tot(U0.abs())
    imp = 0.5 * dt * (tot(U0[0] * st.g1) + tot(st.U1[0] * st.g2))
    work = 0.5 * dt * (tot(U0[1:4] * st.g1).sum() + tot(st.U1[1:4] * st.g2).sum())
    gs = 0.5 * dt * (tot((U0[0] * st.g1).abs()) + tot((st.U1[0] * st.g2).abs()))
    print(json.dumps({"L": L, "step": k, "mass_rel": abs(d[0].item()) / scale[0].item(),
                      "mom_resid_over_impulse_scale": [abs(d[1 + c].item() - imp[c].item())
                                                       / gs[c].item() for c in range(3)],
                      "mom_resid_abs": [abs(d[1 + c].item() - imp[c].item()) for c in range(3)],
                      "energy_resid_rel": abs(d[4].item() - work.item()) / scale[4].item(),
                      "net_momentum": tot(st.U[1:4]).tolist(),
                      "abs_momentum": tot(st.U[1:4].abs()).tolist()}))
