#!/bin/bash
# Long-list search in order of decreasing m: parity (random + full-size tests), then C2 / C5 / C3 bench lines.
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_loopback.py -x -q > gpurun_out/long_pytest.log 2>&1; echo "pytest exit=$?"
B="python bench.py --no-e2e --no-cpu --no-f4 --no-v1"
timeout 300 $B --config C2 --rotations 1 > gpurun_out/long_C2.json 2>gpurun_out/long_C2.err; echo "C2 exit=$?"
timeout 400 $B --config C5 --rotations 1 --steps 10 > gpurun_out/long_C5.json 2>gpurun_out/long_C5.err; echo "C5 exit=$?"
timeout 300 $B --config C3 --rotations 2 > gpurun_out/long_C3.json 2>gpurun_out/long_C3.err; echo "C3 exit=$?"
timeout 300 $B --config C4 --rotations 1 > gpurun_out/long_C4.json 2>gpurun_out/long_C4.err; echo "C4 exit=$?"
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/long_C*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        r = d["roofline"]; s = d.get("stages_ms", {})
        print(f"{f[11:-5]:10s} {d['value']:9.1f} VDIs/s  ms/VDI {r['ms']:.4f}  frac {r['frac']:.3f}  single {r['single_vdi_merge_stage']['ms']:.4f}  fast {s.get('merge_fast', 0):.4f} search {s.get('merge_search', 0):.4f} buckets {d.get('search_buckets')}")
    except Exception as e:
        print(f, "ERR", e)
PY
