#!/bin/bash
# Final build, multi-GPU (gpurun --gpus 4): parity check at G = 2 and 4 (tests/mgpu_check.py), bench lines at
# N = 2 and 4 (strip mode, frames in flight, rotating root and replicas as secondary fields). Outputs gpurun_out/f2m_*.
mkdir -p gpurun_out
for g in 2 4; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $g --master-addr 127.0.0.1 --master-port 2971$g tests/mgpu_check.py > gpurun_out/f2m_check$g.log 2>&1
  echo "check G=$g exit=$?"
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $g --master-addr 127.0.0.1 --master-port 2972$g bench.py --gpus $g --rotating > gpurun_out/f2m_bench_n$g.json 2> gpurun_out/f2m_bench_n$g.err
  echo "bench N=$g exit=$?"
done
