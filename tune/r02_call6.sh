set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/c6_pytest.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/c6_pytest.log
/usr/bin/time -v timeout 900 python bench.py > gpurun_out/c6_bench.json 2> gpurun_out/c6_bench.err; echo bench_rc=$?
tail -25 gpurun_out/c6_bench.err | grep -E "Elapsed|Maximum resident"
timeout 2400 python tools/parity_report.py > gpurun_out/c6_parity_report.json 2> gpurun_out/c6_parity.err; echo parity_rc=$?
tail -8 gpurun_out/c6_parity.err
