set -x
python -c "import __graft_entry__ as g; g.build()"
bash tune/ab3.sh "main variants/libvsr_gs4.so+VSR_ORDER_PROXY=grid variants/libvsr_mix1.so+VSR_ORDER_PROXY=grid variants/libvsr_mix2.so+VSR_ORDER_PROXY=grid" "C2:any C2:closest C4:any C5:any" 2 > gpurun_out/c36_ab.txt 2>&1
cat gpurun_out/c36_ab.txt
