#!/bin/bash
# A/B of (library, env) pairs on bench.py headline lines:
#   tune/ab3.sh "LIB[+NAME=VALUE[,NAME=VALUE]] ..." "CONFIG:QUERY ..." REPS
# LIB is `main` (the in-tree library) or a path (VSR_LIB=path).
LIBS=$1; CASES=$2; R=${3:-2}
for i in $(seq $R); do
  for c in $CASES; do
    CFG=${c%%:*}; Q=${c##*:}
    for LE in $LIBS; do
      L=${LE%%+*}; E=""
      if [ "$LE" != "$L" ]; then E=${LE#*+}; E=${E//,/ }; fi
      if [ "$L" = main ]; then LIBSET=""; else LIBSET="VSR_LIB=$L"; fi
      env $LIBSET $E timeout 600 python bench.py --config $CFG --query $Q --no-variants --no-cpu --no-counters \
        --strong-config none --steps 200 --warmup 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readlines()[-1])
print('$LE', '$CFG', '$Q', d['value'], d['ms_median'], d['roofline']['kernel_ms'])"
    done
  done
done
