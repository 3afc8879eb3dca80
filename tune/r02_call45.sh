set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -q -x > gpurun_out/c45_pytest.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/c45_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c45_smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/c45_smoke.log
timeout 900 python bench.py > gpurun_out/c45_bench.json 2> gpurun_out/c45_bench.err; echo bench_rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/c45_bench.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'], json.dumps(d['cpu_baseline'].get('parity')))"
