#!/bin/bash
# Round-2 final build (after the shared-memory slot rows and the long-search frame schedule):
# GPU suite, bench lines (C3 default with e2e / CPU baseline / f4; C2, C4, C5, C5 with 16 PEs),
# launch list of the timed C3 step, ncu --set full of the C3 merge kernels and of the C5 long search.
# One GPU; outputs gpurun_out/f2_*.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/f2_pytest.log 2>&1; echo "pytest exit=$?"
timeout 600 python bench.py > gpurun_out/f2_bench_n1.json 2> gpurun_out/f2_bench_n1.err; echo "bench exit=$?"
for c in C2 C4; do
  timeout 600 python bench.py --config $c --no-e2e --no-cpu --no-f4 > gpurun_out/f2_bench_$c.json 2> gpurun_out/f2_bench_$c.err; echo "$c exit=$?"
done
timeout 900 python bench.py --config C5 --steps 10 --no-e2e --no-cpu --no-f4 --rotations 2 > gpurun_out/f2_bench_C5.json 2> gpurun_out/f2_bench_C5.err; echo "C5 exit=$?"
timeout 900 python bench.py --config C5 --pes 16 --steps 10 --no-e2e --no-cpu --no-f4 --rotations 1 > gpurun_out/f2_bench_C5-16.json 2> gpurun_out/f2_bench_C5-16.err; echo "C5-16 exit=$?"
K="regex:merge_|search_|long_|chunk_|group_base|general|compact|margins|push|bounds"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" --csv --log-file gpurun_out/f2_launches.csv python bench.py --no-e2e --no-cpu --no-f4 --no-v1 --rotations 1 --steps 3 --warmup 3 > gpurun_out/f2_ncu_launch.log 2>&1; echo "launch list exit=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:merge_fast|search_gather|search_sweep|long_search|merge_general" -s 10 -c 5 -f -o gpurun_out/f2_c3_full python bench.py --no-e2e --no-cpu --no-f4 --no-v1 --rotations 1 --steps 3 --warmup 3 > gpurun_out/f2_ncu_full.log 2>&1; echo "full exit=$?"
timeout 1200 ncu --set full --clock-control none -k "regex:long_search|merge_fast" -c 2 -f -o gpurun_out/f2_c5_full python bench.py --config C5 --no-e2e --no-cpu --no-f4 --no-v1 --rotations 1 --steps 1 --warmup 3 > gpurun_out/f2_ncu_c5.log 2>&1; echo "c5 full exit=$?"
