#!/bin/bash
# Native machine quick A/B: parity tests, the 512 worker sweep, C4 modes,
# the reference-API call at C4 (bench.py legs, compact JSON).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_native_machine.py tests/test_gpu_plugin_path.py -x -q 2>&1 | tail -3
timeout 1200 python - <<'PY'
import json, bench
r = lambda d: {k: (round(v, 3) if isinstance(v, float) else v) for k, v in d.items()
               if not isinstance(v, (dict, str))}
a = bench.machine_ablation()
print("512", json.dumps({k: r(v) for k, v in a.get("workers_sweep", {}).items()}), flush=True)
print("c4", json.dumps(r(bench.machine_ablation_c4())), flush=True)
p = bench.plugin_call_bench()
print("plugin", json.dumps({k: r(v) for k, v in p.items() if isinstance(v, dict)}), flush=True)
PY
