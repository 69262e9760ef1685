#!/bin/bash
# C5 strong-scaling sweep of BASELINE.json configs[4] (3840x2160, k = 32): 2 / 4 / 8 PEs on 1 / 2 / 4 GPUs
# (16 PEs on 8 GPUs needs a box gpurun does not give).  gpurun --gpus 4; outputs gpurun_out/c5s_*.json
B="--config C5 --no-e2e --no-cpu --no-f4 --no-v1 --rotations 1 --steps 10"
timeout 900 python bench.py $B --pes 2 > gpurun_out/c5s_n2_g1.json 2> gpurun_out/c5s_n2_g1.err; echo "pes=2 G=1 exit=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29812 bench.py --gpus 2 $B --pes 4 > gpurun_out/c5s_n4_g2.json 2> gpurun_out/c5s_n4_g2.err; echo "pes=4 G=2 exit=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29814 bench.py --gpus 4 $B --pes 8 > gpurun_out/c5s_n8_g4.json 2> gpurun_out/c5s_n8_g4.err; echo "pes=8 G=4 exit=$?"
timeout 900 python bench.py $B --pes 8 > gpurun_out/c5s_n8_g1.json 2> gpurun_out/c5s_n8_g1.err; echo "pes=8 G=1 exit=$?"
