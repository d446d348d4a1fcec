#!/bin/bash
# The N=2 code path on one GPU (two gloo ranks): default (fused X1), and with the fused
# exchange's probe failing on rank 1 (LIFT_X1_PROBE_FAIL=1): every rank must fall back to NCCL/gloo.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for fail in "" 1; do
LIFT_X1_PROBE_FAIL=$fail LIFT_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 \
  > gpurun_out/bench_n2_$fail.json 2> gpurun_out/bench_n2_$fail.err
echo "n2 fail=$fail rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/bench_n2_$fail.json').read().strip().splitlines()[-1])
print(d['value'], d['config']['x1']); sc=d.get('scaling_configs') or {}
print({k:(v.get('bits_equal_unsharded'), [p for p in ('kernel','fused','nccl') if p in v], v.get('fused')) for k,v in sc.items() if isinstance(v,dict)})"
tail -2 gpurun_out/bench_n2_$fail.err
done
