#!/bin/bash
# Native machine / plugin path: parity tests, the call-phase breakdown and the bench leg.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_native_machine.py tests/test_gpu_plugin_path.py tests/test_gpu_faults.py tests/test_gpu_machinery.py -x -q 2>&1 | tail -3
timeout 300 python scripts/plugin_call_phases.py 3
timeout 600 python -c "
import json, bench
print(json.dumps(bench.plugin_call_bench()))" > gpurun_out/plugin_call.json 2>&1; tail -c 1500 gpurun_out/plugin_call.json
