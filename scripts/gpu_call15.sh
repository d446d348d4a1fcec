#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python scripts/ab.py build/liblift_old3586.so build/liblift_nv_r2u4.so build/liblift_nv_r1u8.so build/liblift_nv_r4u2.so build/liblift_nv_r2u8.so > gpurun_out/ab15.log 2>&1
cat gpurun_out/ab15.log
