"""Does the bench's process context change the C4 machine ablation? C4 leg
standalone, then after the plugin-call leg, then after the 512 ablation;
thread counts of the process at each point."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def threads():
    return len(os.listdir("/proc/self/task"))


def c4(tag):
    d = bench.machine_ablation_c4(steps=4)
    keep = {k: round(v, 2) for k, v in d.items() if isinstance(v, float) and "ms" in k}
    keep["sweep"] = {k: {kk: round(vv, 2) for kk, vv in v.items()} for k, v in d["sweep"].items()}
    print(tag, "threads", threads(), json.dumps(keep), flush=True)


c4("fresh")
c4("fresh-again")
bench.plugin_call_bench()
c4("after-plugin")
bench.machine_ablation()
c4("after-512")
