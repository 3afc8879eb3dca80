set -x
python -c "import __graft_entry__ as g; g.build()"
bash tune/ab2.sh "main env:VSR_SCHED=region" "C2:any C2:closest C5:any C4:any" 3 > gpurun_out/c25_ab.txt 2>&1
cat gpurun_out/c25_ab.txt
VSR_SCHED=region timeout 900 python bench.py --no-variants --strong-config none > gpurun_out/c25_region_any.json 2>gpurun_out/c25_region_any.err
python - <<'P'
import json
d=json.loads(open("gpurun_out/c25_region_any.json").read().strip().splitlines()[-1])
print(d["value"], json.dumps(d["cpu_baseline"].get("parity")))
P
