#!/bin/bash
# First-wave stagger on scal (knob values 1 = off, 0 = auto, 2, 3 ns per 32 KiB): ab.py and the
# bench step, interleaved by process, twice.
cd $GRAFT_REPO_ROOT
for r in 1 2; do for v in 1 0 2 3; do echo "== stagger=$v"; LIFT_SET_VARIANTS=stagger=$v python scripts/ab.py --child 2>/dev/null | python -c "
import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(' '.join(f'{k}:{x[\"us\"]}' for k,x in d.items()))"; done; done
for r in 1 2; do for v in 1 0 2 3; do echo "== step stagger=$v"; LIFT_SET_VARIANTS=stagger=$v timeout 300 python scripts/step_ab.py 20 2>&1 | python -c "
import sys,json; d=json.load(sys.stdin); print({k:v['ms'] for k,v in d.items() if k in ('seq_events','seq_plain')})"; done; done
