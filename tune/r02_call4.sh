set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/c4_pytest.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/c4_pytest.log
bash tune/ab2.sh "main variants/libvsr_ldg128.so" "C2:any C2:closest" 3 > gpurun_out/c4_ab_ldg.txt 2>&1
bash tune/ab2.sh "main variants/libvsr_ldg128.so" "C5:any" 1 >> gpurun_out/c4_ab_ldg.txt 2>&1
for i in 1 2; do for L in main variants/libvsr_instcost0.so variants/libvsr_multi0.so; do
  if [ $L = main ]; then unset VSR_LIB; else export VSR_LIB=$L; fi
  timeout 600 python tune/inst_bench.py 30 >> gpurun_out/c4_inst.txt 2>&1
done; done
unset VSR_LIB
cat gpurun_out/c4_ab_ldg.txt gpurun_out/c4_inst.txt
