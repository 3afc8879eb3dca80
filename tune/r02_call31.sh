set -x
python -c "import __graft_entry__ as g; g.build()"
bash tune/ab2.sh "main env:VSR_OCC=1" "C2:any C2:closest" 3 > gpurun_out/c31_ab.txt 2>&1
cat gpurun_out/c31_ab.txt
python bench.py --probe > /dev/null 2>&1; echo probe=$?
ncu --set full --clock-control none --import-source on -k regex:trace_kernel -s 2 -c 1 -o gpurun_out/r02_c2_any_v3 python bench.py --probe > gpurun_out/ncu_c31.log 2>&1; echo ncu=$?
