#!/bin/bash
# bench lines with the Phase-1 + Phase-2 (volume -> root VDI) stage at N=1 and N=2; outputs in gpurun_out/.
set -x
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 300 python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err
timeout 400 $R --nproc-per-node 2 --master-port 29601 bench.py --gpus 2 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$? >> gpurun_out/smoke.log
