set -x
python -c "import __graft_entry__ as g; g.build()"
export VSR_SCHED=region
python bench.py --probe > /dev/null 2>&1; echo probe=$?
ncu --set full --clock-control none --import-source on -k regex:trace_kernel_region -s 2 -c 1 -o gpurun_out/r02_c2_region python bench.py --probe > gpurun_out/ncu_region.log 2>&1; echo ncu=$?
