set -x
python -c "import __graft_entry__ as g; g.build()"
bash tune/ab2.sh "main variants/libvsr_idsmem.so" "C2:any C2:closest C5:any C4:any" 3 > gpurun_out/c32_ab.txt 2>&1
cat gpurun_out/c32_ab.txt
