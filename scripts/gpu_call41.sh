#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
LIFT_LIB=$PWD/build/liblift_pre.so timeout 600 python -m pytest tests -m gpu -q -x -k gemv > gpurun_out/pytest_pre.log 2>&1; echo "pytest(pre) rc=$?"; tail -1 gpurun_out/pytest_pre.log
timeout 600 python scripts/ab.py build/liblift_base.so build/liblift_pre.so build/liblift_base.so build/liblift_pre.so > gpurun_out/ab41.log 2>&1
python - <<'P'
import json
for line in open('gpurun_out/ab41.log'):
    parts=line.strip().split('} {')
    if len(parts)<2: continue
    lib=json.loads(parts[0]+'}')['lib']; d=json.loads('{'+parts[1].split('}} ')[0]+'}}')
    print(lib, {k: d[k]['GB/s'] for k in ('gemv_8192','gemv_8192x16384')})
P
