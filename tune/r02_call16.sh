set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/c16_pytest.log 2>&1; echo pytest_rc=$?
tail -4 gpurun_out/c16_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c16_smoke.log 2>&1; echo smoke_rc=$?; tail -2 gpurun_out/c16_smoke.log
START=$(date +%s); timeout 900 python bench.py > gpurun_out/c16_bench.json 2> gpurun_out/c16_bench.err; echo bench_rc=$? wall=$(( $(date +%s) - START ))
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/c16_ref.json 2>&1; echo ref_rc=$?
