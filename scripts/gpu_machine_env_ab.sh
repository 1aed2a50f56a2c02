#!/bin/bash
# Native machine A/B over environment knobs: scripts/machine_diag.py under
# each "VAR=value ..." argument (one run of the whole case list per setting).
for setting in "$@"; do
  echo "== $setting"
  env $setting timeout 600 python scripts/machine_diag.py 2>&1 | grep -v '^{"diag"' 
done
