#!/bin/bash
# A/B/C of in-tree builds on one GPU (VDI_LIB_PATH): lib/libvdi_<variant>.so; outputs in gpurun_out/.
set -x
L=$PWD/paper_2206_14503_b200/lib
timeout 300 env VDI_LIB_PATH=$L/libvdi_sp9.so python -m pytest tests -m gpu -x -q -k "parity and not multi" > gpurun_out/ab_sp9_pytest.log 2>&1
for r in 1 2; do
  for c in C3 C2; do
    timeout 300 python bench.py --config $c --no-e2e --no-cpu > gpurun_out/ab_A_${c}_$r.json 2>/dev/null
    for v in sp9 sp10; do
      VDI_LIB_PATH=$L/libvdi_$v.so timeout 300 python bench.py --config $c --no-e2e --no-cpu > gpurun_out/ab_${v}_${c}_$r.json 2>/dev/null
    done
  done
done
