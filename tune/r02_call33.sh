set -x
python -c "import __graft_entry__ as g; g.build()"
for i in 1 2 3; do
for L in main variants/libvsr_scopy.so variants/libvsr_scopy_outer.so; do
  if [ $L = main ]; then unset VSR_LIB; else export VSR_LIB=$L; fi
  timeout 600 python tune/inst_bench.py 30 2>/dev/null | tail -1
done; done
unset VSR_LIB
