"""How the L2 treatment between timed steps changes the measured K2 step at
C4 (32768 sub-grids): write-flush (bench default), read-flush, and steps
back to back (inputs 128 MiB + outputs 128 MiB exceed the 126 MB L2)."""

import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_08058_b200 import _native as N  # noqa: E402
from paper_2303_08058_b200.ring import RingStepper  # noqa: E402

BYTES = 32768 * 512 * 16.28125


def main():
    K = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    N.init(0)
    st = RingStepper(32768, device=torch.device("cuda", 0), max_steps=8 * K + 100)
    for _ in range(10):
        st.step()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    out = {}
    for mode in ("write_flush", "read_flush", "none_per_step", "back_to_back"):
        torch.cuda.synchronize()
        if mode == "back_to_back":
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(K):
                st.step()
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / K
        else:
            evs = []
            for _ in range(K):
                if mode == "write_flush":
                    flush.fill_(1)
                elif mode == "read_flush":
                    flush.sum(dtype=torch.int64)
                k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                st.step(kernel_events=(k0, k1))
                evs.append((k0, k1))
            torch.cuda.synchronize()
            ms = sum(x.elapsed_time(y) for x, y in evs) / K
        out[mode] = {"ms": ms, "frac_of_6548": BYTES / (ms * 1e-3) / 1e9 / 6548.8}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
