#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
LIFT_BENCH_DEBUG=1 LIFT_DIST_BACKEND=gloo timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 5 --warmup 3 --e2e-steps 2 > gpurun_out/bench_n2_gloo.log 2>&1
echo "torchrun rc=$?"; grep -v "^\s" gpurun_out/bench_n2_gloo.log | tail -4 | cut -c1-600
