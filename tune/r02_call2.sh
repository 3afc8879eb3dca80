set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/c2_pytest.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/c2_pytest.log
timeout 900 python bench.py > gpurun_out/c2_bench.json 2> gpurun_out/c2_bench.err; echo bench_rc=$?
tail -3 gpurun_out/c2_bench.err
timeout 900 python bench.py --config C2K --no-variants --no-cpu --strong-config none > gpurun_out/c2_bench_c2k.json 2> gpurun_out/c2_bench_c2k.err; echo c2k_rc=$?
tail -3 gpurun_out/c2_bench_c2k.err
python tune/prof_secondary.py both && \
ncu --set full --clock-control none --import-source on -k regex:trace_instances_kernel -s 2 -c 1 -o gpurun_out/r02_inst python tune/prof_secondary.py instances > gpurun_out/ncu_inst.log 2>&1; echo ncu_inst=$?
ncu --set full --clock-control none --import-source on -k regex:trace_multi_kernel -s 2 -c 1 -o gpurun_out/r02_multi python tune/prof_secondary.py multi > gpurun_out/ncu_multi.log 2>&1; echo ncu_multi=$?
python bench.py --probe && ncu --set full --clock-control none --import-source on -k regex:trace_kernel -s 2 -c 1 -o gpurun_out/r02_c2_any python bench.py --probe > gpurun_out/ncu_c2.log 2>&1; echo ncu_c2=$?
