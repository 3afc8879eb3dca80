set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "knobs or warp" > gpurun_out/c8_pytest.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/c8_pytest.log
bash tune/ab2.sh "main env:VSR_SCHED=warp" "C2:any C2:closest C5:any C4:any" 3 > gpurun_out/c8_ab_warp.txt 2>&1
cat gpurun_out/c8_ab_warp.txt
