set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/c7_pytest.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/c7_pytest.log
START=$(date +%s); timeout 900 python bench.py > gpurun_out/c7_bench.json 2> gpurun_out/c7_bench.err; echo bench_rc=$? wall=$(( $(date +%s) - START ))
bash tune/ab2.sh "main variants/libvsr_sent0.so" "C2:any C5:any" 3 > gpurun_out/c7_ab_sent.txt 2>&1
for i in 1 2; do for L in main variants/libvsr_instminb8.so; do
  if [ $L = main ]; then unset VSR_LIB; else export VSR_LIB=$L; fi
  timeout 600 python tune/inst_bench.py 30 >> gpurun_out/c7_inst.txt 2>&1
done; done
unset VSR_LIB
cat gpurun_out/c7_ab_sent.txt gpurun_out/c7_inst.txt
