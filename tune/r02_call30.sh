set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "ragged or knobs" > gpurun_out/c30_pytest.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/c30_pytest.log
for L in main variants/libvsr_multiouter.so main variants/libvsr_multiouter.so main variants/libvsr_multiouter.so; do
  if [ $L = main ]; then unset VSR_LIB; else export VSR_LIB=$L; fi
  timeout 600 python tune/multi_bench.py 2>/dev/null | tail -1 | sed "s|^|$L |"
done
unset VSR_LIB
