#!/bin/bash
# Round-2 final bench lines of the other configs (1 GPU): C2, C4, C5 (8 PEs), C5 with 16 PEs.  Outputs gpurun_out/r2_bench_<cfg>.json
for c in C2 C4; do
  timeout 600 python bench.py --config $c --no-e2e --no-cpu --no-f4 > gpurun_out/r2_bench_$c.json 2> gpurun_out/r2_bench_$c.err; echo "$c exit=$?"
done
timeout 900 python bench.py --config C5 --steps 10 --no-e2e --no-cpu --no-f4 --rotations 2 > gpurun_out/r2_bench_C5.json 2> gpurun_out/r2_bench_C5.err; echo "C5 exit=$?"
timeout 900 python bench.py --config C5 --pes 16 --steps 10 --no-e2e --no-cpu --no-f4 --rotations 1 > gpurun_out/r2_bench_C5-16.json 2> gpurun_out/r2_bench_C5-16.err; echo "C5-16 exit=$?"
