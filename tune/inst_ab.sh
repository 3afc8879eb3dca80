#!/bin/bash
# A/B of library builds on the bench's instanced / multi-hit extras: tune/inst_ab.sh REPS LIB...
R=$1; shift
for i in $(seq $R); do
  for L in "$@"; do
    VSR_LIB=$L python bench.py --no-cpu --steps 50 --warmup 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readlines()[-1])
print('$L', 'instanced', d['instanced']['value'], d['instanced']['ms'], 'multi', d['multi_hit']['value'], 'head', d['value'])"
  done
done
