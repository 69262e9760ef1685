#!/bin/bash
# Last check of the round: GPU suite, smoke(), default bench line (one GPU). Outputs gpurun_out/last_*.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/last_pytest.log 2>&1; echo "pytest exit=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/last_smoke.log 2>&1; echo "smoke exit=$?"
timeout 600 python bench.py > gpurun_out/last_bench.json 2> gpurun_out/last_bench.err; echo "bench exit=$?"
