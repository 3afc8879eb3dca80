set -x
python -c "import __graft_entry__ as g; g.build()"
bash tune/ab2.sh "main variants/libvsr_mix8.so variants/libvsr_mixw.so" "C2:any C2:closest C4:any C5:any" 2 > gpurun_out/c44_ab.txt 2>&1
cat gpurun_out/c44_ab.txt
