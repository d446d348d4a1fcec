#!/bin/bash
# racecheck of every kernel path (sanitize_probe.py) + the TMA-ring gemv variant's parity tests.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python scripts/sanitize_probe.py > gpurun_out/san_racecheck.log 2>&1
echo "racecheck rc=$?"; tail -3 gpurun_out/san_racecheck.log
timeout 600 python -m pytest tests/test_gpu_variants.py -q -x 2>&1 | tail -1
AB_SHAPES=8192x8192,4096x4096 AB_VARS=0,3 python scripts/gemv_xs_ab.py --child 2>&1 >/dev/null
