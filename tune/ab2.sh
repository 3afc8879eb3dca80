#!/bin/bash
# A/B of library builds / runtime knobs on bench.py headline lines:
#   tune/ab2.sh "LIBS" "CONFIG:QUERY ..." REPS
# a LIB is `main` (the in-tree library), a path (VSR_LIB=path) or env:NAME=VALUE (a knob).
LIBS=$1; CASES=$2; R=${3:-2}
for i in $(seq $R); do
  for c in $CASES; do
    CFG=${c%%:*}; Q=${c##*:}
    for L in $LIBS; do
      unset VSR_LIB
      ENVSET=""
      if [ "${L:0:4}" = "env:" ]; then ENVSET="${L:4}"; elif [ "$L" != main ]; then export VSR_LIB=$L; fi
      env $ENVSET timeout 600 python bench.py --config $CFG --query $Q --no-variants --no-cpu --no-counters \
        --strong-config none --steps 200 --warmup 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readlines()[-1])
print('$L', '$CFG', '$Q', d['value'], d['ms_median'], d['roofline']['kernel_ms'])"
    done
  done
done
unset VSR_LIB
