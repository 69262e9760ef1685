#!/bin/bash
# ncu evidence of the round-2 final build (1 GPU, C3): the launch list of the timed step and one
# --set full capture of the merge kernels.  Outputs gpurun_out/r2f_launches.csv, gpurun_out/r2f_c3_full.ncu-rep
K="regex:merge_|search_|long_|chunk_|group_base|general|compact|margins|push|bounds"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" --csv --log-file gpurun_out/r2f_launches.csv python bench.py --no-e2e --no-cpu --no-f4 --no-v1 --rotations 1 --steps 3 --warmup 3 > gpurun_out/r2f_ncu_launch.log 2>&1; echo "launch list exit=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:merge_fast|search_gather|search_sweep|long_search|merge_general" -s 10 -c 5 -f -o gpurun_out/r2f_c3_full python bench.py --no-e2e --no-cpu --no-f4 --no-v1 --rotations 1 --steps 3 --warmup 3 > gpurun_out/r2f_ncu_full.log 2>&1; echo "full exit=$?"
