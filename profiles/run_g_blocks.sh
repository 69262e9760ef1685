#!/bin/bash
# NVLink push block budgets (VDI_XBLOCKS exchange push, VDI_GBLOCKS gather compaction) vs frames-in-flight
# ms per VDI at G = $1 ranks (profiles/frames_probe.py).  Outputs gpurun_out/gb_*.txt
G=${1:-2}
port=29600
for xb in 1184 296 148; do for gb in 1184 296 148; do
  port=$((port+1))
  VDI_XBLOCKS=$xb VDI_GBLOCKS=$gb timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G --master-addr 127.0.0.1 --master-port $port profiles/frames_probe.py > gpurun_out/gb_G${G}_x${xb}_g${gb}.txt 2>/dev/null
  echo "G=$G x=$xb g=$gb $(tail -1 gpurun_out/gb_G${G}_x${xb}_g${gb}.txt | cut -c1-330)"
done; done
