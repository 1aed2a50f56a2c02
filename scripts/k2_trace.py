"""Per-step trace of K2 at the driver's bench command shape (C4, 20 timed
steps after 5 warm-up steps): where does a short timed window lose time
against the long back-to-back runs? Phases, each on a fresh idle gap or not,
with NVML SM-clock samples every ~0.5 ms tagged by phase. Output: one JSON
document (profiles/r02/k2_trace.json)."""
import json
import os
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_08058_b200 import _native as N  # noqa: E402
from paper_2303_08058_b200.ring import RingStepper, run_reference_gpu  # noqa: E402


def main():
    out_path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/k2_trace.json"
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    samples = []
    stop = threading.Event()

    def loop():
        while not stop.is_set():
            t = time.perf_counter()
            try:
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
            except Exception:  # noqa: BLE001
                continue
            samples.append((t, time.perf_counter(), sm, rs))
            time.sleep(0.0005)

    th = threading.Thread(target=loop, daemon=True)
    th.start()
    dev = torch.device("cuda", 0)
    N.init(0)
    run_reference_gpu(512, 15, device=dev)
    st = RingStepper(32768, device=dev, max_steps=8000)
    res = {"phases": []}

    def phase(name, steps, per_step=False, gap_s=0.0):
        torch.cuda.synchronize()
        if gap_s:
            time.sleep(gap_s)
        t0 = time.perf_counter()
        if per_step:
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
            ev[0].record()
            for i in range(steps):
                st.step()
                ev[i + 1].record()
            torch.cuda.synchronize()
            per = [ev[i].elapsed_time(ev[i + 1]) * 1e3 for i in range(steps)]
            tot = ev[0].elapsed_time(ev[-1]) * 1e3
        else:
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(steps):
                st.step()
            b.record()
            torch.cuda.synchronize()
            per = None
            tot = a.elapsed_time(b) * 1e3
        t1 = time.perf_counter()
        sm = [s for (ta, tb, s, _) in samples if ta >= t0 - 0.002 and tb <= t1 + 0.002]
        res["phases"].append({"name": name, "steps": steps, "us_per_step": tot / steps,
                              "per_step_us": per, "gap_s": gap_s, "wall_s": t1 - t0,
                              "sm_mhz_samples": sm})

    for _ in range(5):          # the bench's warm-up
        st.step()
    phase("bench_replica_20", 20, gap_s=0.05)
    phase("per_step_20", 20, per_step=True)
    phase("b2b_3000", 3000)
    phase("after_warm_20", 20)
    phase("after_warm_per_step_20", 20, per_step=True)
    phase("idle_0.5s_20", 20, gap_s=0.5)
    phase("idle_0.5s_per_step_40", 40, per_step=True, gap_s=0.5)
    phase("idle_2s_per_step_40", 40, per_step=True, gap_s=2.0)
    # time-based warm-up policy: >= 200 ms of steps, then 20 timed
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    n = 0
    while time.perf_counter() - t0 < 0.2:
        for _ in range(50):
            st.step()
        torch.cuda.synchronize()
        n += 50
    phase("warm200ms_then_20", 20)
    res["warm_steps"] = n
    stop.set()
    th.join()
    res["all_samples"] = [(round(ta, 5), s, rs) for (ta, _, s, rs) in samples[::4]]
    os.makedirs(os.path.dirname(out_path) or ".", exist_ok=True)
    with open(out_path, "w") as fh:
        json.dump(res, fh)
    for p in res["phases"]:
        sm = p["sm_mhz_samples"]
        print(f"{p['name']:28s} {p['us_per_step']:8.2f} us/step  clocks "
              f"{min(sm) if sm else None}-{max(sm) if sm else None} n={len(sm)}"
              + (f"  per-step {[round(x, 1) for x in p['per_step_us'][:12]]}"
                 if p["per_step_us"] else ""))


if __name__ == "__main__":
    main()
