#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) over the
# 1-GPU parity tests of small configurations and the loopback (G = 2, 3, 4)
# device path.  Run from the repo root under gpurun; logs in gpurun_out/.
make -s >/dev/null 2>&1
SEL='merge_parity_random or empty_and_transparent or composite_frames_one_gpu or loopback_strips or loopback_composite_frames or limit_case_c1'
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --target-processes all --print-limit 50 --error-exitcode 99 \
    python -m pytest tests -m gpu -q -p no:cacheprovider -k "$SEL" > gpurun_out/sanitizer_$tool.log 2>&1
  echo "exit=$?" >> gpurun_out/sanitizer_$tool.log
done
