#!/bin/bash
# Round-end check on one GPU: clean build, full GPU test suite, smoke, default bench; outputs in gpurun_out/.
set -x
make clean >/dev/null 2>&1; make -s > gpurun_out/final_build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/final_pytest.log 2>&1; echo rc=$? >> gpurun_out/final_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo rc=$? >> gpurun_out/final_smoke.log
timeout 300 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err
