#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -k gemv > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python scripts/ab.py build/liblift_r2u4.so build/liblift_r1u8.so build/liblift_r2u2.so build/liblift_r4u2.so build/liblift_r1u4.so build/liblift_r2u6.so > gpurun_out/ab13.log 2>&1
cat gpurun_out/ab13.log
