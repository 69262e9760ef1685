#!/bin/bash
# Round-2 measurements behind profiles/r2_*: bench lines (C3 default, C2, C4,
# C5, C5 with 16 PEs), the launch list of the timed step, ncu --set full of the
# merge kernels (C3) and of the long-list search (C5).  Run from the repo root
# under gpurun (one GPU); outputs land in gpurun_out/.
set -x
make -s >/dev/null 2>&1
timeout 600 python bench.py > gpurun_out/r2_bench_n1.json 2> gpurun_out/r2_bench_n1.err
for c in C2 C4; do
  timeout 600 python bench.py --config $c --no-e2e --no-cpu --no-f4 > gpurun_out/r2_bench_$c.json 2> gpurun_out/r2_bench_$c.err
done
timeout 900 python bench.py --config C5 --steps 10 --no-e2e --no-cpu --no-f4 --rotations 2 > gpurun_out/r2_bench_C5.json 2> gpurun_out/r2_bench_C5.err
timeout 900 python bench.py --config C5 --pes 16 --steps 10 --no-e2e --no-cpu --no-f4 --rotations 1 > gpurun_out/r2_bench_C5-16.json 2> gpurun_out/r2_bench_C5-16.err
K="regex:merge_|search_|long_|chunk_|group_base|general|compact|margins|push|bounds"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" --csv --log-file gpurun_out/r2_launches.csv python bench.py --no-e2e --no-cpu --no-f4 --no-v1 --rotations 1 --steps 3 --warmup 3 > gpurun_out/r2_ncu_launch.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:merge_fast|search_gather|search_sweep|long_search|merge_general" -s 10 -c 5 -o gpurun_out/r2_c3_full python bench.py --no-e2e --no-cpu --no-f4 --no-v1 --rotations 1 --steps 3 --warmup 3 > gpurun_out/r2_ncu_full.log 2>&1
timeout 1200 ncu --set full --clock-control none -k "regex:long_search|merge_fast" -c 2 -o gpurun_out/r2_c5_full python bench.py --config C5 --no-e2e --no-cpu --no-f4 --no-v1 --rotations 1 --steps 1 --warmup 3 > gpurun_out/r2_ncu_c5.log 2>&1
