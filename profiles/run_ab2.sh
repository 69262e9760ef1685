#!/bin/bash
# Generic A/B on one GPU: parity tests on the default build, then bench lines per config and build.
#   VARIANTS="gold pol" CONFIGS="C3 C2" REPS=2 bash profiles/run_ab2.sh
# builds: default (paper_2206_14503_b200/lib/libvdi.so) and build_ab/libvdi_<variant>.so; outputs gpurun_out/ab2_*.json
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_loopback.py -x -q > gpurun_out/ab2_pytest.log 2>&1; echo "pytest exit=$?"
B="python bench.py --no-e2e --no-cpu --no-f4 --no-v1"
for r in $(seq 1 ${REPS:-1}); do
for c in ${CONFIGS:-C3}; do
  X="--rotations 2"; [ $c = C5 ] && X="--rotations 1 --steps 10"
  timeout 400 $B --config $c $X > gpurun_out/ab2_${c}_base_$r.json 2>/dev/null; echo "$c base $?"
  for v in $VARIANTS; do VDI_LIB_PATH=$PWD/build_ab/libvdi_$v.so timeout 400 $B --config $c $X > gpurun_out/ab2_${c}_${v}_$r.json 2>/dev/null; echo "$c $v $?"; done
done
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/ab2_C*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        r = d["roofline"]; s = d.get("stages_ms", {})
        print(f"{f[15:-5]:14s} {d['value']:9.1f} VDIs/s  ms/VDI {r['ms']:.4f}  frac {r['frac']:.3f}  single {r['single_vdi_merge_stage']['ms']:.4f}  fast {s.get('merge_fast', 0):.4f} search {s.get('merge_search', 0):.4f}")
    except Exception as e:
        print(f, "ERR", e)
PY
