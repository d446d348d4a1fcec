#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python scripts/ab.py build/liblift_base.so build/liblift_np16.so build/liblift_np8.so build/liblift_np4.so build/liblift_np4f32.so build/liblift_g1u8.so build/liblift_g1u8np.so build/liblift_g2u4np.so build/liblift_g1u4.so > gpurun_out/ab3.log 2>&1
cat gpurun_out/ab3.log
