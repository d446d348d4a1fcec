#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fuzz.py -q > gpurun_out/pytest_fuzz.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_fuzz.log
tail -5 gpurun_out/pytest_fuzz.log
LIFT_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 5 --warmup 3 --e2e-steps 2 > gpurun_out/bench_n2_gloo.log 2>&1
echo "torchrun rc=$?"; tail -5 gpurun_out/bench_n2_gloo.log
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"; cat gpurun_out/bench_ref.log
