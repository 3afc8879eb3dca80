set -x
python -c "import __graft_entry__ as g; g.build()"
for P in len grid; do VSR_ORDER_PROXY=$P VSR_LIB=variants/lib_timeline.so QUERY=any OUT=gpurun_out/timeline_$P.npy timeout 300 python tools/timeline.py > gpurun_out/c14_timeline_$P.txt 2>&1; head -13 gpurun_out/c14_timeline_$P.txt; done
bash tune/ab2.sh "main env:VSR_ORDER_PROXY=grid" "C2:any C2:closest C4:any C5:any" 3 > gpurun_out/c14_ab_grid.txt 2>&1
cat gpurun_out/c14_ab_grid.txt
