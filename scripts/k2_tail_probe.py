"""K2 back to back at C4: the fused-finalize step (tb_step_final) and the
deferred one (tb_step_deferred, the bench's launch) vs the step without the accumulator (tb_step, acc = NULL) vs with the
accumulator but no finalize: what the exact checksum and its last-CTA
rounding cost per step."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_08058_b200 import _native as N  # noqa: E402


def main():
    K = 300
    N.init(0)
    n = 32768
    dev = torch.device("cuda", 0)
    st = [torch.empty((n, 512), dtype=torch.float64, device=dev) for _ in range(2)]
    s = torch.cuda.current_stream().cuda_stream
    N.call("tb_init_cells", s, st[0].data_ptr(), n, 0, n)
    acc = torch.zeros(N.TB_ACC_WORDS, dtype=torch.int64, device=dev)
    N.call("tb_acc_reset", s, acc.data_ptr())
    ds = torch.zeros((2, n), dtype=torch.float64, device=dev)
    dm = torch.zeros((2, n), dtype=torch.float64, device=dev)
    sacc = torch.zeros(N.TB_ACC_WORDS, dtype=torch.int64, device=dev)
    out = torch.zeros(3, dtype=torch.float64, device=dev)
    res = {}
    for mode in ("final", "no_acc", "sums_only", "deferred") * 3:
        def launch(k):
            o, w = st[k & 1], st[(k + 1) & 1]
            lf, rf = o[-1, -8:].data_ptr(), o[0, :8].data_ptr()
            if mode == "final":
                N.call("tb_step_final", s, o.data_ptr(), w.data_ptr(), n, lf, rf, 3, 5, None,
                       None, acc.data_ptr(), out[0:1].data_ptr(), out[1:2].data_ptr(),
                       out[2:3].data_ptr())
            elif mode == "deferred":
                N.call("tb_step_deferred", s, o.data_ptr(), w.data_ptr(), n, lf, rf, 3, 5,
                       ds[k & 1].data_ptr(), dm[k & 1].data_ptr(),
                       ds[(k - 1) & 1].data_ptr() if k else None,
                       dm[(k - 1) & 1].data_ptr() if k else None, sacc.data_ptr(),
                       out[0:1].data_ptr(), out[1:2].data_ptr(), out[2:3].data_ptr())
            elif mode == "sums_only":
                N.call("tb_step", s, o.data_ptr(), w.data_ptr(), n, lf, rf, 3, 5,
                       dm[k & 1].data_ptr(), ds[k & 1].data_ptr(), None)
            elif mode == "acc_only":
                N.call("tb_step", s, o.data_ptr(), w.data_ptr(), n, lf, rf, 3, 5, None, None,
                       acc.data_ptr())
            else:
                N.call("tb_step", s, o.data_ptr(), w.data_ptr(), n, lf, rf, 3, 5, None, None,
                       None)
        for k in range(10):
            launch(k)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for k in range(K):
            launch(k)
        b.record()
        torch.cuda.synchronize()
        res.setdefault(mode, []).append(round(a.elapsed_time(b) / K * 1e3, 2))
        if mode == "acc_only":
            N.call("tb_acc_reset", s, acc.data_ptr())
    print(json.dumps({"us_per_step": res}))


if __name__ == "__main__":
    main()
