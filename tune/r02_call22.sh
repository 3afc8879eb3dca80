set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/c22_pytest.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/c22_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/c22_smoke.log 2>&1; echo smoke_rc=$?; tail -2 gpurun_out/c22_smoke.log
timeout 900 python bench.py > gpurun_out/c22_bench.json 2> gpurun_out/c22_bench.err; echo bench_rc=$?; tail -c 600 gpurun_out/c22_bench.json
