#!/bin/bash
# Round-2 multi-GPU measurements (gpurun --gpus 4): the parity check at G = 2
# and 4, bench lines at N = 2 and 4 (strip mode, frames in flight, single and
# rotating root), the frames probe.  Outputs in gpurun_out/.
make -s >/dev/null 2>&1
for g in 2 4; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $g --master-addr 127.0.0.1 --master-port 2951$g tests/mgpu_check.py > gpurun_out/r2_mgpu$g.log 2>&1
  echo "rc=$?" >> gpurun_out/r2_mgpu$g.log
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $g --master-addr 127.0.0.1 --master-port 2952$g bench.py --gpus $g --rotating > gpurun_out/r2_bench_n$g.json 2> gpurun_out/r2_bench_n$g.err
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $g --master-addr 127.0.0.1 --master-port 2953$g profiles/frames_probe.py > gpurun_out/r2_probe$g.json 2> gpurun_out/r2_probe$g.err
done
