#!/bin/bash
# occupancy variant: auto (default) vs VSR_OCC=0 / 1: [Q=any] tune/occ_ab.sh CONFIG
CFG=$1; QQ=${Q:-closest}
for O in auto 0 1; do
  if [ $O = auto ]; then unset VSR_OCC; else export VSR_OCC=$O; fi
  python bench.py --config $CFG --query $QQ --no-variants --no-cpu --steps 100 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readlines()[-1])
print('occ=$O', '$CFG', '$QQ', d['value'], d['ms_median'], d['roofline']['kernel_ms'])"
done
