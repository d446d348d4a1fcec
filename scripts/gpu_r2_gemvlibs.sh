#!/bin/bash
# gemv shapes: in-tree build vs build/var_*.so (gemv_xs_ab.py per library, auto variant), twice.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export AB_SHAPES=${AB_SHAPES:-1024x8192,512x8192,2048x8192,4096x4096,2048x4096,8192x8192}
LIBS=${LIBS:-"paper_1502_02389_b200/liblift.so $(ls build/var_*.so)"}
for r in 1 2; do for l in $LIBS; do echo "== $l"; LIFT_LIB=$PWD/$l AB_VARS=${AB_VARS:-0} python scripts/gemv_xs_ab.py --child 2>&1 >/dev/null | python -c "
import sys,json
for l in sys.stdin:
    k,d=l.split(' ',1); d=json.loads(d); print(k, ' '.join(f'{v}:{d[v][\"us\"]}' for v in d if v.startswith('v')), d['same_bits'])"; done; done
