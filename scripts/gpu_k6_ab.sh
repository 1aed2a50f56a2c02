#!/bin/bash
# K6 A/B: bit-exactness tests + config-2 timing for each TB_HYDRO_VARIANT given.
mkdir -p gpurun_out
for v in "$@"; do
  echo "== variant $v"
  TB_HYDRO_VARIANT=$v timeout 600 python -m pytest tests/test_gpu_hydro.py -x -q 2>&1 | tail -2
  for S in ${SIZES:-4096 32768}; do
    TB_HYDRO_VARIANT=$v timeout 300 python scripts/bench_hydro.py $S 30 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('v$v', $S, round(d['ms'],4), 'fp64_frac', round($S*321408/(d['ms']*1e-3)/18.543e12,3))"
  done
done
