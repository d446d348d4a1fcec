#!/bin/bash
# Round evidence: GPU tests, bench (default args), ncu launch list + full captures.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=${TAG:-r1}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
tail -2 gpurun_out/${TAG}_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?"; cat gpurun_out/${TAG}_bench.json
timeout 600 python scripts/sweep.py > gpurun_out/${TAG}_sweep.json 2> gpurun_out/${TAG}_sweep.err
TAG=$TAG bash scripts/profile_round.sh
