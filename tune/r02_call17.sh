set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_instances.py -q -x > gpurun_out/c17_pytest.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/c17_pytest.log
for i in 1 2 3; do
  timeout 600 python tune/inst_bench.py 30 >> gpurun_out/c17_inst.txt 2>&1
  VSR_ORDER_PROXY=grid timeout 600 python tune/inst_bench.py 30 | sed 's/^default/grid/' >> gpurun_out/c17_inst.txt 2>&1
done
cat gpurun_out/c17_inst.txt
