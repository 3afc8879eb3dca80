set -x
python -c "import __graft_entry__ as g; g.build()"
bash tune/ab2.sh "main env:VSR_ORDER_PROXY=grid" "C2:any C2:closest C4:any C5:any" 3 > gpurun_out/c15_ab_grid.txt 2>&1
cat gpurun_out/c15_ab_grid.txt
