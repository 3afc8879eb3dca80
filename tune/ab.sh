#!/bin/bash
# A/B of two library builds on one box: alternate runs, print value + kernel_ms.
# usage: tune/ab.sh LIB_A LIB_B CONFIG QUERY [ISECT] [REPS]
A=$1; B=$2; CFG=$3; Q=$4; IS=${5:-alpha_texture}; R=${6:-3}
for i in $(seq $R); do
  for L in $A $B; do
    VSR_LIB=$L python bench.py --config $CFG --query $Q --isect $IS --no-variants --no-cpu \
      --steps 200 --warmup 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readlines()[-1])
print('$L', '$CFG', '$Q', d['value'], d['ms_median'], d['roofline']['kernel_ms'])"
  done
done
