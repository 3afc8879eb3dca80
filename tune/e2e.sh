#!/bin/bash
# e2e (vsr_trace_host) per chunk size: tune/e2e.sh CONFIG QUERY SIZES...  ("default": unset)
CFG=$1; Q=$2; shift 2
for c in "$@"; do
  if [ "$c" = default ]; then unset VSR_HOST_CHUNK; else export VSR_HOST_CHUNK=$c; fi
  python bench.py --config $CFG --query $Q --no-variants --no-cpu --steps 50 --warmup 5 \
    2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readlines()[-1]); e=d['e2e']
print('chunk', '$c', 'tail', '${VSR_HOST_TAIL:-1}', '$CFG', '$Q', 'e2e', e['value'], e.get('ms_per_step'), 'kernel-path', d['value'])"
done
