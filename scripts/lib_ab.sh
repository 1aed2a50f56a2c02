#!/bin/bash
# Same-box A/B of two libtb builds: runs the given python script under each
# library (TB_LIBTB), alternating, $REPS times. usage: lib_ab.sh A.so B.so script [args]
A=$1; B=$2; shift 2
for r in $(seq ${REPS:-2}); do
  for lib in $A $B; do
    echo "== $lib"
    TB_LIBTB=$lib timeout 900 python "$@"
  done
done
