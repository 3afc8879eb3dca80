set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_wide.py -x -q > gpurun_out/c5_pytest_wide.log 2>&1; echo wide_rc=$?
tail -15 gpurun_out/c5_pytest_wide.log
for c in C2:any C2:closest C5:any C5:closest C4:any; do
  CFG=${c%%:*}; Q=${c##*:}
  for B in binary wide; do
    timeout 900 python bench.py --config $CFG --query $Q --bvh $B --no-variants --no-cpu --no-counters --strong-config none --steps 100 > gpurun_out/c5_${CFG}_${Q}_${B}.json 2>&1
    python -c "
import json; d=json.loads(open('gpurun_out/c5_${CFG}_${Q}_${B}.json').read().strip().splitlines()[-1]); print('$CFG $Q $B', d['value'], d['ms_median'], d['roofline']['kernel_ms'], d['config'].get('wide_bvh'))"
  done
done
python bench.py --probe --bvh wide && ncu --set full --clock-control none --import-source on -k regex:trace_wide_kernel -s 2 -c 1 -o gpurun_out/r02_c2_any_wide python bench.py --probe --bvh wide > gpurun_out/ncu_wide.log 2>&1; echo ncu=$?
