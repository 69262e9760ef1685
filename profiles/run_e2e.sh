#!/bin/bash
# e2e pipeline check on one GPU: parity tests, bench C3 (24 and 48 frames); outputs in gpurun_out/.
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_e2e.log 2>&1
timeout 300 python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err
timeout 300 python bench.py --e2e-steps 48 --no-cpu --steps 20 > gpurun_out/bench_n1_e48.json 2> gpurun_out/bench_n1_e48.err
