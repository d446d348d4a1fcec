#!/bin/bash
# gemv C4-shape knob sweep: stagger values with the L2 prefetch on (auto) and off.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export AB_SHAPES=${AB_SHAPES:-8192x8192,16384x8192,8192x12288,16384x4096}
for pf in 0 1; do echo "== prefetch=$pf"; LIFT_SET_VARIANTS=prefetch=$pf AB_KNOB=stagger AB_VARS=1,2,3,4,5 python scripts/gemv_xs_ab.py --child 2>&1 >/dev/null | python -c "
import sys,json
for l in sys.stdin:
    k,d=l.split(' ',1); d=json.loads(d); print(k, ' '.join(f'{v}:{d[v][\"us\"]}' for v in d if v.startswith('v')), d['same_bits'])"; done
