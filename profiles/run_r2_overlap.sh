#!/bin/bash
# Round-2 experiments (1 GPU): frames-in-flight overlap knobs on C3 (search stream
# priority, search share, pass-through residency) and the long-search residency
# (VDI_LONG_WPS builds) on C2 / C5.  Outputs: gpurun_out/ov_*.json
B="python bench.py --no-e2e --no-cpu --no-f4 --no-v1"
run() { name=$1; shift; env "$@" timeout 300 $B $EXTRA > gpurun_out/ov_$name.json 2> gpurun_out/ov_$name.err; echo "$name exit=$?"; }
EXTRA="--config C3 --rotations 2"
for r in 1 2; do
run c3_base_$r X=1
run c3_prio_hi_$r VDI_SST_PRIO=1
run c3_prio_lo_$r VDI_SST_PRIO=-1
run c3_share375_$r VDI_SEARCH_SHARE=0.375
run c3_share375_fw9_$r VDI_SEARCH_SHARE=0.375 VDI_FAST_WARPS=9
run c3_fw8_$r VDI_FAST_WARPS=8
run c3_hi_share5_$r VDI_SST_PRIO=1 VDI_SEARCH_SHARE=0.5
done
EXTRA="--config C2 --rotations 1"
run c2_base X=1
run c2_w4 VDI_LIB_PATH=$PWD/build_ab/libvdi_w4.so
run c2_w6 VDI_LIB_PATH=$PWD/build_ab/libvdi_w6.so
EXTRA="--config C5 --rotations 1 --steps 10"
run c5_base X=1
run c5_w4 VDI_LIB_PATH=$PWD/build_ab/libvdi_w4.so
run c5_w6 VDI_LIB_PATH=$PWD/build_ab/libvdi_w6.so
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/ov_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        r = d["roofline"]; s = d.get("stages_ms", {})
        print(f"{f[14:-5]:24s} {d['value']:9.1f} VDIs/s  ms/VDI {r['ms']:.4f}  frac {r['frac']:.3f}  single {r['single_vdi_merge_stage']['ms']:.4f}  fast {s.get('merge_fast', 0):.4f} search {s.get('merge_search', 0):.4f}")
    except Exception as e:
        print(f, "ERR", e)
PY
