#!/bin/bash
# Multi-GPU bench lines (gpurun --gpus 4): N = 2 and 4, strip mode with 4 frames in flight per GPU, rotating root
# and replicas as secondary fields.  Outputs gpurun_out/r2_bench_n{2,4}.json
for g in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $g --master-addr 127.0.0.1 --master-port 2962$g bench.py --gpus $g --rotating > gpurun_out/r2_bench_n$g.json 2> gpurun_out/r2_bench_n$g.err
  echo "N=$g exit=$?"
done
