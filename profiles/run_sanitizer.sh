#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over smoke() (the C1-sized composite of __graft_entry__,
# 3840 lists: pass-through, short and long search, general path) and one small loopback test. Logs gpurun_out/san_*.
mkdir -p gpurun_out
S="python -c 'import __graft_entry__ as g; g.smoke(); print(\"smoke ok\")'"
for t in memcheck racecheck synccheck initcheck; do
  timeout 420 compute-sanitizer --tool $t --print-limit 30 --error-exitcode 9 bash -c "$S" > gpurun_out/san_$t.log 2>&1
  echo "$t exit=$?"
done
timeout 600 compute-sanitizer --tool memcheck --print-limit 30 --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x -k "merge_parity_random or composite_parity_c1_oracle_inputs or empty_and_transparent" > gpurun_out/san_memcheck_parity.log 2>&1
echo "memcheck parity exit=$?"
