#!/bin/bash
# A/B/n of library builds on one box: tune/abn.sh CONFIG QUERY ISECT REPS LIB...
CFG=$1; Q=$2; IS=$3; R=$4; shift 4
for i in $(seq $R); do
  for L in "$@"; do
    VSR_LIB=$L python bench.py --config $CFG --query $Q --isect $IS --no-variants --no-cpu \
      --steps 200 --warmup 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readlines()[-1])
print('$L', '$CFG', '$Q', d['value'], d['ms_median'], d['roofline']['kernel_ms'])"
  done
done
