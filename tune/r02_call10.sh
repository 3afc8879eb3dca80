set -x
python -c "import __graft_entry__ as g; g.build()"
for Q in any closest; do VSR_LIB=variants/lib_timeline.so QUERY=$Q OUT=gpurun_out/timeline_$Q.npy timeout 300 python tools/timeline.py > gpurun_out/c10_timeline_$Q.txt 2>&1; echo rc=$?; cat gpurun_out/c10_timeline_$Q.txt; done
