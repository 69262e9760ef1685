#!/bin/bash
# The GPU-box commands behind profiles/r1_v18_*: launch list, ncu --set full
# of the top kernels, bench lines of the other configs.  Run from the repo root
# under gpurun; outputs land in gpurun_out/.
set -x
make -s >/dev/null 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "host_dense" > gpurun_out/pytest_hd.log 2>&1
timeout 300 python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err
K="regex:merge_|search_|long_|chunk_|group_base|general|compact|peer_copy"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" --csv --log-file gpurun_out/launches_v18.csv python bench.py --no-e2e --no-cpu --steps 3 --warmup 3 > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:merge_fast|search_gather|search_sweep" -s 6 -c 3 -o gpurun_out/v18_full python bench.py --no-e2e --no-cpu --steps 3 --warmup 3 > gpurun_out/ncu_full.log 2>&1
timeout 300 python bench.py --config C4 > gpurun_out/bench_C4.json 2>gpurun_out/bench_C4.err
timeout 300 python bench.py --config C5 --steps 20 > gpurun_out/bench_C5.json 2>gpurun_out/bench_C5.err
timeout 300 python bench.py --config C2 > gpurun_out/bench_C2.json 2>gpurun_out/bench_C2.err
