#!/bin/bash
# Machine parity tests + host-side diagnostics (512 worker sweep, C4 gather,
# C4 resident at E8/E16), one log.
timeout 900 python -m pytest tests/test_gpu_native_machine.py tests/test_gpu_plugin_path.py -x -q 2>&1 | tail -2
timeout 600 python scripts/machine_diag.py 2>&1
for a in "16 8 256" "16 16 256"; do timeout 300 python scripts/machine_diag_c4.py $a 2>&1; done
