#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python scripts/sweep.py > gpurun_out/sweep29.json 2> gpurun_out/sweep29.err; echo "sweep rc=$?"
python - <<'P'
import json; d=json.load(open('gpurun_out/sweep29.json'))
for k,v in d.items():
    if k!='note': print(k, v['us'], v['GB/s'])
P
