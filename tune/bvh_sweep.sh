#!/bin/bash
# BVH build parameter sweep: tune/bvh_sweep.sh CONFIG "LEAF:BINS ..."
CFG=$1; shift
for lb in $@; do
  L=${lb%%:*}; B=${lb##*:}
  python bench.py --config $CFG --no-variants --no-cpu --max-leaf $L --sah-bins $B --steps 100 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readlines()[-1]); w=d['roofline']['work_per_ray']
print('$CFG leaf $L bins $B', d['value'], d['ms_median'], d['roofline']['kernel_ms'], round(w['inner_per_ray'],2), round(w['tris_per_ray'],2), d['config']['setup_s'])"
done
