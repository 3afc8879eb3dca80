#!/bin/bash
# A/B of the 1-bit alpha plane (VSR_ALPHA_BITS=1 default vs 0): tune/bits_ab.sh CONFIG QUERY REPS
CFG=$1; Q=$2; R=$3
for i in $(seq $R); do
  for B in 1 0; do
    VSR_ALPHA_BITS=$B python bench.py --config $CFG --query $Q --no-variants --no-cpu \
      --steps 200 --warmup 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readlines()[-1])
print('bits=$B', '$CFG', '$Q', d['value'], d['ms_median'], d['roofline']['kernel_ms'])"
  done
done
