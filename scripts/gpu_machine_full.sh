#!/bin/bash
# Full GPU suite + criteria 4/5 numbers + the machine legs of the bench line.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_ablation.py tests/test_gpu_native_machine.py::test_native_polling_beats_fence -q -s 2>&1 | grep -E "speedup|vs|passed|failed" | head
timeout 600 python -c "
import json, bench
print(json.dumps(bench.plugin_call_bench()))" > gpurun_out/plugin_call.json 2>&1; tail -c 1200 gpurun_out/plugin_call.json
