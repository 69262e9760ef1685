#!/bin/bash
# Short-sweep sample residency A/B (VDI_SWEEP_R samples in registers, the rest in shared memory):
# parity on the default build, then C3 / C2 bench values per build.  Outputs: gpurun_out/sw_*.json
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > gpurun_out/sw_pytest.log 2>&1; echo "pytest exit=$?"
B="python bench.py --no-e2e --no-cpu --no-f4 --no-v1 --rotations 2"
run() { name=$1; shift; env "$@" timeout 300 $B $EXTRA > gpurun_out/sw_$name.json 2> gpurun_out/sw_$name.err; echo "$name exit=$?"; }
for r in 1 2; do
for c in C3 C2; do
EXTRA="--config $c"
run ${c}_r16_$r X=1
for v in r24 r8 r16m14 r40; do run ${c}_${v}_$r VDI_LIB_PATH=$PWD/build_ab/libvdi_$v.so; done
done
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/sw_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        r = d["roofline"]; s = d.get("stages_ms", {})
        print(f"{f[14:-5]:18s} {d['value']:9.1f} VDIs/s  ms/VDI {r['ms']:.4f}  frac {r['frac']:.3f}  single {r['single_vdi_merge_stage']['ms']:.4f}  fast {s.get('merge_fast', 0):.4f} search {s.get('merge_search', 0):.4f}  parity {d.get('parity_sample', {}).get('count_mismatches')}")
    except Exception as e:
        print(f, "ERR", e)
PY
