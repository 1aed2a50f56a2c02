#!/bin/bash
# The paper's Tests 1 and 2 figure structure on the native
# machine: per integration (host task = Test 1, event polling = Test 2) and
# its fence twin ("integration off"), (1) executors 1..128 without
# aggregation at 16 workers, (2) one executor with aggregation 1..64, (3) the
# best combination E32 M8 over workers 1..8. 512 sub-grids, 6 steps, median
# of 3 repeats; staged batches (the reference's H2D ; kernel ; D2H) and the
# B200 direct batches.
OUT=${OUT:-gpurun_out/paper}
mkdir -p $OUT
for zc in off direct; do
  for I in hosttask polling; do
    for S in executors aggregation workers; do
      timeout 900 python -m paper_2303_08058_b200.cli --engine native --zero-copy $zc \
        --integration $I --sweep $S --workers 16 --executors 32 --max-agg 8 --subgrids 512 \
        --steps 6 --repeats 3 --output csv --out $OUT/${zc}_${I}_${S}.csv > $OUT/${zc}_${I}_${S}.log 2>&1
      echo "$zc $I $S rc=$?"
    done
  done
done
