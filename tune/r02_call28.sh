set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_fuzz.py tests/test_gpu_alpha_bits.py tests/test_gpu_variants.py -m gpu -q -x > gpurun_out/c28_pytest.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/c28_pytest.log
timeout 900 python bench.py > gpurun_out/c28_bench.json 2> gpurun_out/c28_bench.err; echo bench_rc=$?
python - <<'P'
import json
d=json.loads(open("gpurun_out/c28_bench.json").read().strip().splitlines()[-1])
print(d["value"], d["ms_per_step"], d["roofline"]["frac"], d["roofline"].get("kernel_ms"), json.dumps(d["cpu_baseline"].get("parity")))
P
