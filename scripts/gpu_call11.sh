#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python scripts/ab.py build/liblift_pair.so > gpurun_out/ab11.log 2>&1
cat gpurun_out/ab11.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gemv_tma" -s 1 -c 1 -o gpurun_out/r1c_gemv python scripts/ncu_probe.py 2 > gpurun_out/r1c_ncu.log 2>&1
echo "ncu rc=$?"
