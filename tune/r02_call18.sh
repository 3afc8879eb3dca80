set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/c18_pytest.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/c18_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c18_smoke.log 2>&1; echo smoke_rc=$?
START=$(date +%s); timeout 900 python bench.py > gpurun_out/c18_bench.json 2> gpurun_out/c18_bench.err; echo bench_rc=$? wall=$(( $(date +%s) - START ))
timeout 900 python bench.py --config C4 --query closest --isect count_alpha_texture --no-variants --no-cpu --strong-config none > gpurun_out/c18_bench_C4_count.json 2>&1; echo rc=$?
