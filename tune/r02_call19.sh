set -x
python -c "import __graft_entry__ as g; g.build()"
bash tune/ab2.sh "main env:VSR_CARVEOUT=0 env:VSR_CARVEOUT=50" "C2:any C5:any" 3 > gpurun_out/c19_ab.txt 2>&1
cat gpurun_out/c19_ab.txt
