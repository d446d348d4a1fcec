#!/bin/bash
# One gpurun call: GPU tests, the N=1 bench line, and an N=2 run of the multi-rank code
# path on the one GPU (gloo transport; its numbers are meaningless, the JSON is checked).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
if [ -z "$SKIP_TESTS" ]; then
timeout ${TEST_TIMEOUT:-1500} python -m pytest tests -m gpu -q -x ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
fi
timeout 900 python bench.py --steps ${STEPS:-50} --warmup 5 --cpu-budget ${CPU_BUDGET:-5} > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"; cut -c1-1500 gpurun_out/bench.json; tail -3 gpurun_out/bench.err
if [ -z "$SKIP_N2" ]; then
LIFT_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 \
  > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err
echo "bench n2 rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/bench_n2.json').read().strip().splitlines()[-1])
print(json.dumps(d.get('scaling_configs'))[:3000])"
tail -3 gpurun_out/bench_n2.err
fi
