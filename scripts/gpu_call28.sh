#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 600 python -m pytest tests -m gpu -q -k gemv > gpurun_out/pytest_gemv.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gemv.log
timeout 600 python scripts/ab.py build/liblift_nopf.so build/liblift_pf.so build/liblift_nopf.so build/liblift_pf.so > gpurun_out/ab28.log 2>&1
cat gpurun_out/ab28.log
