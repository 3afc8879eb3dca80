set -x
python -c "import __graft_entry__ as g; g.build()"
python bench.py --probe --query closest > /dev/null 2>&1; echo probe=$?
ncu --set full --clock-control none --import-source on -k regex:trace_kernel -s 2 -c 1 -o gpurun_out/r02_c2_closest_v4 python bench.py --probe --query closest > gpurun_out/ncu_c39.log 2>&1; echo ncu=$?
