#!/bin/bash
# Mid-size reductions: in-tree build vs build/var_*.so, interleaved twice (midsize_ab.py).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
LIBS=${LIBS:-"paper_1502_02389_b200/liblift.so $(ls build/var_*.so)"}
for r in 1 2; do for l in $LIBS; do echo "== $l"; LIFT_LIB=$PWD/$l timeout 300 python scripts/midsize_ab.py; done; done
