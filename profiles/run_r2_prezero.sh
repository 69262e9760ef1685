#!/bin/bash
# Zero fill + records-only pass-through (default) vs the pass-through writing zeros (VDI_PREZERO=0):
# GPU tests, the frames timeline (trace_probe.py), bench lines on C3 / C4 / C2.
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pz_pytest.log 2>&1; echo "pytest exit=$?"
timeout 300 python profiles/trace_probe.py C3 4 > gpurun_out/pz_trace_c3.txt 2>&1; echo "trace exit=$?"
B="python bench.py --no-e2e --no-cpu --no-f4 --no-v1 --rotations 2"
for c in C3 C4 C2; do
  timeout 400 $B --config $c > gpurun_out/pz_${c}_on.json 2>/dev/null; echo "$c on $?"
  VDI_PREZERO=0 timeout 400 $B --config $c > gpurun_out/pz_${c}_off.json 2>/dev/null; echo "$c off $?"
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/pz_C*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        r = d["roofline"]; s = d.get("stages_ms", {})
        print(f"{f[14:-5]:10s} {d['value']:9.1f} VDIs/s  ms/VDI {r['ms']:.4f}  frac {r['frac']:.3f}  single {r['single_vdi_merge_stage']['ms']:.4f}  fast {s.get('merge_fast', 0):.4f} search {s.get('merge_search', 0):.4f} parity {d.get('parity_sample', {}).get('count_mismatch')}")
    except Exception as e:
        print(f, "ERR", e)
PY
