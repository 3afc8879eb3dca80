set -x
python -c "import __graft_entry__ as g; g.build()"
START=$(date +%s); timeout 900 python bench.py > gpurun_out/c9_bench.json 2> gpurun_out/c9_bench.err; echo bench_rc=$? wall=$(( $(date +%s) - START ))
timeout 900 python bench.py --query closest --no-cpu --strong-config none > gpurun_out/c9_bench_C2_closest.json 2>&1; echo rc=$?
timeout 900 python bench.py --config C4 --query closest --isect count_alpha_texture --no-variants --no-cpu --strong-config none > gpurun_out/c9_bench_C4_count.json 2>&1; echo rc=$?
timeout 900 python bench.py --config C4 --no-variants --no-cpu --strong-config none > gpurun_out/c9_bench_C4_any.json 2>&1; echo rc=$?
timeout 900 python bench.py --config C5 --no-variants --no-cpu --strong-config none > gpurun_out/c9_bench_C5_any.json 2>&1; echo rc=$?
timeout 900 python bench.py --config C5 --query closest --no-variants --no-cpu --strong-config none > gpurun_out/c9_bench_C5_closest.json 2>&1; echo rc=$?
timeout 900 python bench.py --config C2K --no-variants --no-cpu --strong-config none > gpurun_out/c9_bench_C2K.json 2>&1; echo rc=$?
python bench.py --steps 3 --warmup 3 --no-cpu --no-counters --strong-config none --no-variants > gpurun_out/c9_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_c2_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-counters --strong-config none --no-variants > gpurun_out/c9_ncu_launches.log 2>&1; echo launches=$?
python bench.py --probe && ncu --set full --clock-control none --import-source on -k regex:trace_kernel -s 2 -c 1 -o gpurun_out/r02_c2_any_final python bench.py --probe > gpurun_out/ncu_final.log 2>&1; echo ncu=$?
python bench.py --probe --query closest && ncu --set full --clock-control none --import-source on -k regex:trace_kernel -s 2 -c 1 -o gpurun_out/r02_c2_closest_final python bench.py --probe --query closest > gpurun_out/ncu_final2.log 2>&1; echo ncu2=$?
