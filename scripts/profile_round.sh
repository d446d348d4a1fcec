#!/bin/bash
# ncu evidence for profiles/: (1) launch list of the bench command (cold-cache, serialised
# per-launch times: compare SHARES), (2) one --set full capture per kernel of the step.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=${TAG:-r2}
mkdir -p gpurun_out
# skip the 7 generator fills + warm-up (3 steps x 4 launches) = 19 launches
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -s 19 -c 40 --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-extras > gpurun_out/${TAG}_ncu_bench.log 2>&1
echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"reduce_kernel|gemv_kernel|scal_kernel" -s 4 -c 4 -o gpurun_out/${TAG}_full \
  python scripts/ncu_probe.py 2 > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "ncu full rc=$?"
