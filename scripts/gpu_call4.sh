#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -4 gpurun_out/pytest_gpu.log
timeout 900 python scripts/ab.py build/liblift_g2u4.so build/liblift_g1u8.so build/liblift_g1u4.so build/liblift_g2u2.so build/liblift_g4u2.so build/liblift_f32.so > gpurun_out/ab4.log 2>&1
cat gpurun_out/ab4.log
timeout 600 python bench.py --steps 100 --warmup 5 --cpu-budget 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
