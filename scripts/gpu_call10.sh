#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -k "gemv" > gpurun_out/pytest_gemv.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gemv.log
tail -3 gpurun_out/pytest_gemv.log
timeout 900 python scripts/ab.py build/liblift_ru1d2.so build/liblift_ru1d4.so build/liblift_ru2d2.so build/liblift_ru2d3.so build/liblift_ru4d2.so build/liblift_ru8d2.so > gpurun_out/ab10.log 2>&1
cat gpurun_out/ab10.log
timeout 600 python bench.py --steps 100 --warmup 5 --cpu-budget 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
