set -x
python -c "import __graft_entry__ as g; g.build()"
bash tune/ab2.sh "main variants/libvsr_keepid.so" "C2:any C2:closest C5:any" 3 > gpurun_out/c20_ab.txt 2>&1
cat gpurun_out/c20_ab.txt
