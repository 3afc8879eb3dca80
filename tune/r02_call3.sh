set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/c3_pytest.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/c3_pytest.log
for i in 1 2; do timeout 600 python bench.py --no-variants --no-cpu --strong-config none > gpurun_out/c3_bench_$i.json 2> gpurun_out/c3_bench_$i.err; echo bench_rc=$?; done
timeout 600 python bench.py --query closest --no-variants --no-cpu --strong-config none --no-counters > gpurun_out/c3_bench_closest.json 2>&1; echo closest_rc=$?
timeout 900 python bench.py --config C5 --no-variants --no-cpu --strong-config none --no-counters > gpurun_out/c3_bench_c5.json 2>&1; echo c5_rc=$?
