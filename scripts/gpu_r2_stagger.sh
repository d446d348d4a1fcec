#!/bin/bash
# A/B of the first-wave stagger (runtime knob LIFT_VAR_STAGGER): reductions (ab.py,
# midsize_ab.py), gemv shapes (gemv_xs_ab.py, interleaved in one process) and the bench step.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
VALS=${VALS:-"1 0 2 4 6"}
for r in 1 2; do for v in $VALS; do echo "== stagger=$v"; LIFT_SET_VARIANTS=stagger=$v python scripts/ab.py --child 2>/dev/null | python -c "
import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(' '.join(f'{k}:{x[\"us\"]}' for k,x in d.items()))"; done; done
for r in 1 2; do for v in $VALS; do echo "== midsize stagger=$v"; LIFT_SET_VARIANTS=stagger=$v python scripts/midsize_ab.py; done; done
AB_KNOB=stagger AB_VARS=$(echo $VALS | tr ' ' ',') AB_SHAPES=${AB_SHAPES:-8192x8192,16384x8192,4096x4096,8192x16384,1024x8192,2048x8192,8192x2048} python scripts/gemv_xs_ab.py --child 2>&1 >/dev/null
for r in 1 2; do for v in $VALS; do echo "== step stagger=$v"; LIFT_SET_VARIANTS=stagger=$v timeout 300 python scripts/step_ab.py 20 2>&1 | python -c "
import sys,json; d=json.load(sys.stdin); print({k:v['ms'] for k,v in d.items() if k in ('seq_events','seq_plain')})"; done; done
