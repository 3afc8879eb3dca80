set -x
python -c "import __graft_entry__ as g; g.build()"
python bench.py --probe > /dev/null 2>&1; echo probe=$?
ncu --set full --clock-control none --import-source on -k regex:trace_kernel -s 2 -c 1 -o gpurun_out/r02_c2_any_v4 python bench.py --probe > gpurun_out/ncu_c38.log 2>&1; echo ncu=$?
