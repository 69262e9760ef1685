#!/bin/bash
# Memory-safety checks in place of compute-sanitizer (closed on this GPU pool):
# the VDI_CHECKS debug build (make debug -> build_dbg/libvdi.so) bounds-checks
# every record / slot / region index the kernels compute from the inputs and
# traps on a violation; the whole -m gpu suite (parity against the oracle,
# loopback groups, f4, full sizes) runs on it.  VDI_FLAG_VALIDATE tests
# (tests/test_gpu_validate.py) check the input validation on the normal build.
# Run from the repo root under gpurun; logs in gpurun_out/.
make -s all debug >/dev/null 2>&1
python -m pytest tests/test_gpu_validate.py -x -q > gpurun_out/validate.log 2>&1; echo "validate exit=$?"
VDI_LIB_PATH=$PWD/build_dbg/libvdi.so timeout 1200 python -m pytest tests -m gpu -q -x --durations=15 \
  > gpurun_out/checks.log 2>&1; echo "checks exit=$?"
