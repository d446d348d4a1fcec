#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
LIFT_LIB=$PWD/build/liblift_clc.so timeout 600 python -m pytest tests -m gpu -q -x -k "asum or dot or fused or fuzz or integer or determinism or sharded" > gpurun_out/pytest_clc.log 2>&1; echo "pytest(clc) rc=$?"; tail -2 gpurun_out/pytest_clc.log
timeout 600 python scripts/ab.py build/liblift_hw.so build/liblift_clc.so build/liblift_hw.so build/liblift_clc.so > gpurun_out/ab38.log 2>&1; cat gpurun_out/ab38.log
