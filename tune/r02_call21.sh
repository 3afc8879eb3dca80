set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_wide.py -q -x > gpurun_out/c21_pytest.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/c21_pytest.log
for c in C2:closest C2:any C5:closest; do CFG=${c%%:*}; Q=${c##*:}
  timeout 900 python bench.py --config $CFG --query $Q --bvh wide --no-variants --no-cpu --no-counters --strong-config none --steps 100 > gpurun_out/c21_${CFG}_${Q}_wide.json 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/c21_${CFG}_${Q}_wide.json').read().strip().splitlines()[-1]); print('$CFG $Q wide', d['value'], d['ms_median'], d['roofline']['kernel_ms'])"
done
