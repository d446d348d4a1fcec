#!/bin/bash
# Cluster-mode reductions (LIFT_RED_CLUSTER builds in build/var_cl*.so): parity tests through
# each build, then ab.py / midsize_ab.py / step_ab.py against the in-tree build.
# (The cluster-mode kernel code was measured slower and not kept in the tree.)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for l in build/var_cl*.so; do
  LIFT_LIB=$PWD/$l timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused.py -q -x 2>&1 | tail -1 | sed "s|^|$l |"
done
SKIP_TESTS=1 bash scripts/gpu_r2_fin.sh
