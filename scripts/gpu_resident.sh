#!/bin/bash
# zero_copy = 3 (device-resident rounds): parity tests + the plugin-call leg at C4.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_native_machine.py tests/test_gpu_plugin_path.py -x -q 2>&1 | tail -3
timeout 600 python -c "
import json, bench
print(json.dumps(bench.plugin_call_bench()))" > gpurun_out/plugin_call.json 2>&1; tail -c 2500 gpurun_out/plugin_call.json
