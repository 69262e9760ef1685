#!/bin/bash
# Long search with L2 eviction priorities (VDI_LONG_POLICY 1: slots evict_last + sources / outputs evict_first;
# 2: slots evict_last only) vs default, on C2 and C5.
timeout 600 env VDI_LIB_PATH=$PWD/build_ab/libvdi_pol.so python -m pytest tests/test_gpu_parity.py -x -q -k "merge_parity" > gpurun_out/pol_pytest.log 2>&1; echo "pytest exit=$?"
B="python bench.py --no-e2e --no-cpu --no-f4 --no-v1 --rotations 1"
for c in C2 C5; do
  X=""; [ $c = C5 ] && X="--steps 10"
  timeout 400 $B --config $c $X > gpurun_out/pol_${c}_base.json 2>/dev/null; echo "$c base $?"
  for v in pol pol2; do VDI_LIB_PATH=$PWD/build_ab/libvdi_$v.so timeout 400 $B --config $c $X > gpurun_out/pol_${c}_$v.json 2>/dev/null; echo "$c $v $?"; done
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/pol_C*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        r = d["roofline"]; s = d.get("stages_ms", {})
        print(f"{f[15:-5]:10s} {d['value']:9.1f} VDIs/s  ms/VDI {r['ms']:.4f}  frac {r['frac']:.3f}  single {r['single_vdi_merge_stage']['ms']:.4f}  fast {s.get('merge_fast', 0):.4f} search {s.get('merge_search', 0):.4f}")
    except Exception as e:
        print(f, "ERR", e)
PY
