#!/bin/bash
# e2e A/B on one box: A = lib/libvdi.so, B = lib/libvdi_e0.so (VDI_E2E_MAPPED=0); outputs in gpurun_out/.
set -x
L=$PWD/paper_2206_14503_b200/lib
python profiles/pcie_probe.py > gpurun_out/pcie2.json 2>&1
for r in 1 2 3; do
  timeout 300 python bench.py --no-cpu --steps 20 > gpurun_out/e2e_A_$r.json 2>/dev/null
  VDI_LIB_PATH=$L/libvdi_e0.so timeout 300 python bench.py --no-cpu --steps 20 > gpurun_out/e2e_B_$r.json 2>/dev/null
done
