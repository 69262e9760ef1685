mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_loopback.py -x -q > gpurun_out/g2_loop.log 2>&1; echo loop=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 tests/mgpu_check.py > gpurun_out/g2_mgpu.log 2>&1; echo mgpu=$?
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29542 profiles/trace_probe_mgpu.py C3 4 rot > gpurun_out/trace_g2rot.txt 2>&1; echo trace=$?
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29543 profiles/frames_probe.py > gpurun_out/g2_frames.txt 2>&1; echo frames=$?
