#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
LIFT_BENCH_DEBUG=1 LIFT_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 4 --steps 3 --warmup 3 --e2e-steps 1 --no-extras > gpurun_out/bench_n4_gloo.log 2>&1
echo "torchrun rc=$?"; grep -v "^\s" gpurun_out/bench_n4_gloo.log | grep -v rank | tail -2 | cut -c1-300
grep -o '"x1": "[^"]*"' gpurun_out/bench_n4_gloo.log
LIFT_X1=nccl LIFT_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --steps 3 --warmup 3 --e2e-steps 1 --no-extras > gpurun_out/bench_n2_x1nccl.log 2>&1
echo "torchrun(x1=nccl path, gloo transport) rc=$?"; grep -o '"x1": "[^"]*"' gpurun_out/bench_n2_x1nccl.log
