set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_instances.py tests/test_gpu_configs.py -m gpu -q -x > gpurun_out/c37_pytest.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/c37_pytest.log
bash tune/ab2.sh "main env:VSR_ORDER_PROXY=len" "C2:any C2:closest C4:any C5:any C5:closest" 2 > gpurun_out/c37_ab.txt 2>&1
cat gpurun_out/c37_ab.txt
timeout 600 python tune/inst_bench.py 30 2>/dev/null | tail -1
