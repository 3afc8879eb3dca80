set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python tune/diag_warp.py 40000 2>&1 | tee gpurun_out/c29_diag.txt
bash tune/ab2.sh "main variants/libvsr_sidepf.so" "C2:any C5:any" 3 > gpurun_out/c29_ab.txt 2>&1
cat gpurun_out/c29_ab.txt
