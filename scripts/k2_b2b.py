"""K2 steps back to back (no flush), for an ncu --cache-control none capture
of one launch in the middle: does the previous step's output stay in L2?"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_08058_b200 import _native as N  # noqa: E402
from paper_2303_08058_b200.ring import RingStepper  # noqa: E402

N.init(0)
st = RingStepper(32768, device=torch.device("cuda", 0), max_steps=100)
for _ in range(40):
    st.step()
torch.cuda.synchronize()
