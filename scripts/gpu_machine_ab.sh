#!/bin/bash
# Native machine A/B over TB_PUSH_SPREAD_MIN (0 = 2W+1 default, 1 = always, 1e9 = never).
for sp in "0" "1" "1000000000"; do
  echo "== spread_min=$sp"
  TB_PUSH_SPREAD_MIN=$sp timeout 600 python -c "
import json, bench
a = bench.machine_ablation()
c = bench.machine_ablation_c4()
print(json.dumps({'512': {k: round(v, 2) for k, v in a.items() if 'ms' in k or 'speed' in k},
                  'c4': {k: round(v, 2) for k, v in c.items() if 'ms' in k or 'speed' in k or 'batch' in k}}))
"
done
