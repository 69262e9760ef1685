mkdir -p gpurun_out
./build_ab/write_probe > gpurun_out/write_probe.txt 2>&1
VARIANTS="nowp" CONFIGS="C3 C2" REPS=2 bash profiles/run_ab2.sh > gpurun_out/ab_wp.txt 2>&1
