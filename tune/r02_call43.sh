set -x
python -c "import __graft_entry__ as g; g.build()"
for P in mix len; do VSR_ORDER_PROXY=$P VSR_LIB=variants/lib_timeline.so QUERY=any OUT=gpurun_out/timeline_$P.npy timeout 300 python tools/timeline.py > gpurun_out/c43_timeline_$P.txt 2>&1; echo rc=$?; head -12 gpurun_out/c43_timeline_$P.txt; done
