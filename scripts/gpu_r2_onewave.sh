#!/bin/bash
# One-wave gemv shapes with the whole grid staggered (build/var_ow.so, LIFT_STAGGER_ONEWAVE):
# stagger knob values, interleaved in one process.
# (The LIFT_STAGGER_ONEWAVE switch was measured slower and not kept in the tree.)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export AB_SHAPES=${AB_SHAPES:-1024x8192,512x8192,2048x8192,4096x4096,2048x4096,8192x2048}
LIFT_LIB=$PWD/build/var_ow.so AB_KNOB=stagger AB_VARS=1,2,4,6,8,12 python scripts/gemv_xs_ab.py --child 2>&1 >/dev/null | python -c "
import sys,json
for l in sys.stdin:
    k,d=l.split(' ',1); d=json.loads(d); print(k, ' '.join(f'{v}:{d[v][\"us\"]}' for v in d if v.startswith('v')), d['same_bits'])"
