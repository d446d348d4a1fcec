#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python scripts/sanitize_probe.py > gpurun_out/san_plain.log 2>&1; echo "plain rc=$?"; tail -1 gpurun_out/san_plain.log
for t in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python scripts/sanitize_probe.py > gpurun_out/san_$t.log 2>&1
  echo "$t rc=$?"; tail -3 gpurun_out/san_$t.log
done
