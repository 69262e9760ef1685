#!/bin/bash
# Multi-GPU bench lines (driver's torchrun launch); outputs in gpurun_out/.
set -x
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 400 $R --nproc-per-node 2 --master-port 29601 bench.py --gpus 2 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err
timeout 400 $R --nproc-per-node 4 --master-port 29602 bench.py --gpus 4 > gpurun_out/bench_n4.json 2> gpurun_out/bench_n4.err
timeout 600 python -m pytest tests -m gpu -x -q -k multi_gpu > gpurun_out/pytest_mgpu.log 2>&1
