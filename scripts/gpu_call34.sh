#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1800 python scripts/tune.py measure gpurun_out/tuning_r1b.json > gpurun_out/tune34.log 2>&1
tail -50 gpurun_out/tune34.log | grep -v '^ '
