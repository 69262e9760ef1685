#!/bin/bash
# Balanced exchange push (every block on every slice, last-block signal): loopback GPU tests, parity check at
# G = 2 and 4, bench lines at N = 2 and 4 (gpurun --gpus 4). Outputs gpurun_out/pb_*.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_loopback.py tests/test_gpu_edges.py -q -x > gpurun_out/pb_loopback.log 2>&1; echo "loopback exit=$?"
for g in 2 4; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $g --master-addr 127.0.0.1 --master-port 2981$g tests/mgpu_check.py > gpurun_out/pb_check$g.log 2>&1
  echo "check G=$g exit=$?"
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $g --master-addr 127.0.0.1 --master-port 2982$g bench.py --gpus $g --rotating > gpurun_out/pb_bench_n$g.json 2> gpurun_out/pb_bench_n$g.err
  echo "bench N=$g exit=$?"
done
