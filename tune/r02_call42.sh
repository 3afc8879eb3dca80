set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 2400 python tools/parity_report.py > gpurun_out/c42_parity_report.json 2> gpurun_out/c42_parity.err; echo parity_rc=$?
tail -8 gpurun_out/c42_parity.err
