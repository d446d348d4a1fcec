#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python scripts/ab.py build/liblift_old3586.so build/liblift_r2u4.so build/liblift_old3586.so build/liblift_r2u4.so build/liblift_r4u2.so > gpurun_out/ab14.log 2>&1
cat gpurun_out/ab14.log
