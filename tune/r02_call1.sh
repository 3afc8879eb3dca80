set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/c1_pytest.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/c1_pytest.log
timeout 600 python bench.py > gpurun_out/c1_bench.json 2> gpurun_out/c1_bench.err; echo bench_rc=$?
timeout 300 python tools/sanitize_gpu.py > gpurun_out/c1_san_plain.log 2>&1 && \
timeout 900 compute-sanitizer --tool memcheck --print-limit 50 python tools/sanitize_gpu.py > gpurun_out/c1_memcheck.log 2>&1; echo memcheck_rc=$?
tail -5 gpurun_out/c1_memcheck.log
