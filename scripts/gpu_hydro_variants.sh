#!/bin/bash
# K6 schedule variants (TB_HYDRO_VARIANT): bit-exactness tests + config-2 timing each.
mkdir -p gpurun_out
for v in ${VARIANTS:-0 1 2 3}; do
  echo "== variant $v"
  TB_HYDRO_VARIANT=$v timeout 600 python -m pytest tests/test_gpu_hydro.py -x -q 2>&1 | tail -1
  for S in 4096 32768; do
    for rep in 1 2; do
      TB_HYDRO_VARIANT=$v timeout 300 python scripts/bench_hydro.py $S 30 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('v$v', $S, round(d['ms'],4))"
    done
  done
done
