set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/c41_pytest.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/c41_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c41_smoke.log 2>&1; echo smoke_rc=$?
START=$(date +%s); timeout 900 python bench.py > gpurun_out/c41_bench.json 2> gpurun_out/c41_bench.err; echo bench_rc=$? wall=$(( $(date +%s) - START ))
timeout 900 python bench.py --query closest --no-cpu --strong-config none > gpurun_out/c41_bench_C2_closest.json 2>&1; echo rc=$?
timeout 900 python bench.py --config C4 --query closest --isect count_alpha_texture --no-variants --no-cpu --strong-config none > gpurun_out/c41_bench_C4_count.json 2>&1; echo rc=$?
timeout 900 python bench.py --config C4 --no-variants --no-cpu --strong-config none > gpurun_out/c41_bench_C4_any.json 2>&1; echo rc=$?
timeout 900 python bench.py --config C5 --no-variants --no-cpu --strong-config none > gpurun_out/c41_bench_C5_any.json 2>&1; echo rc=$?
timeout 900 python bench.py --config C5 --query closest --no-variants --no-cpu --strong-config none > gpurun_out/c41_bench_C5_closest.json 2>&1; echo rc=$?
timeout 900 python bench.py --config C2K --no-variants --no-cpu --strong-config none > gpurun_out/c41_bench_C2K.json 2>&1; echo rc=$?
timeout 900 python bench.py --impl reference > gpurun_out/c41_ref.json 2>&1; echo ref_rc=$?
