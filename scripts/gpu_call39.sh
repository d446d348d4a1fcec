#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"reduce_kernel|blackscholes" -s 2 -c 2 -o gpurun_out/r1_next python scripts/ncu_probe_next.py > gpurun_out/r1_next.log 2>&1; echo "ncu rc=$?"
timeout 300 python -m pytest tests/test_abi.py -m gpu -q > gpurun_out/cex.log 2>&1; echo "cex rc=$?"; tail -2 gpurun_out/cex.log
