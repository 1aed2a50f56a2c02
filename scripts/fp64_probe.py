"""Measure the B200's FP64 issue rate (DADD, DMUL, DFMA, DMUL+DADD pairs) with
tb_fp64_probe and print one JSON object: the FP64 roofline denominator used in
DESIGN.md (MEASURED_PEAKS.json has only HBM and bf16 numbers)."""

import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_08058_b200 import _native as N  # noqa: E402


def main():
    N.init(0)
    sms = N.sm_count(0)
    out = {"sms": sms}
    for name, op in (("dadd", N.TB_PROBE_DADD), ("dmul", N.TB_PROBE_DMUL),
                     ("dfma", N.TB_PROBE_DFMA), ("dmul_dadd", N.TB_PROBE_DMUL_DADD)):
        best = 0.0
        mhz = ctypes.c_double()
        for _ in range(3):
            r = ctypes.c_double()
            N.call("tb_fp64_probe", op, 1 << 16, ctypes.byref(r), ctypes.byref(mhz))
            best = max(best, r.value)
        out[name + "_instr_per_s"] = best
        out[name + "_per_sm_per_clk_at_max"] = best / sms / (mhz.value * 1e6)
    out["nominal_sm_mhz"] = mhz.value
    out["dfma_tflops"] = 2 * out["dfma_instr_per_s"] / 1e12
    print(json.dumps(out))


if __name__ == "__main__":
    main()
