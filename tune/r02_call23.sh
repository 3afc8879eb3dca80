set -x
python -c "import __graft_entry__ as g; g.build()"
bash tune/ab2.sh "main variants/libvsr_spec.so" "C2:any C2:closest C5:any C5:closest C4:any" 3 > gpurun_out/c23_ab.txt 2>&1
cat gpurun_out/c23_ab.txt
VSR_LIB=variants/libvsr_spec.so timeout 900 python bench.py --no-variants --strong-config none > gpurun_out/c23_spec_any.json 2>gpurun_out/c23_spec_any.err
VSR_LIB=variants/libvsr_spec.so timeout 900 python bench.py --query closest --no-variants --strong-config none > gpurun_out/c23_spec_closest.json 2>gpurun_out/c23_spec_closest.err
python - <<'P'
import json
for f in ["c23_spec_any","c23_spec_closest"]:
    d=json.loads(open(f"gpurun_out/{f}.json").read().strip().splitlines()[-1])
    print(f, d["value"], json.dumps(d["cpu_baseline"].get("parity")))
P
