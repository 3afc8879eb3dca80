set -x
python -c "import __graft_entry__ as g; g.build()"
python bench.py --steps 3 --warmup 3 --no-cpu --no-counters --strong-config none --no-variants > gpurun_out/c40_plain.log 2>&1; echo plain=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_c2_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-counters --strong-config none --no-variants > gpurun_out/c40_ncu_launches.log 2>&1; echo launches=$?
