#!/bin/bash
# A/B of the reductions' completion schemes: in-tree build vs build/var_*.so (ab.py, midsize_ab.py, step_ab.py).
# (Used for the designated-finisher, next-wave-prefetch and tagged-partial experiments, whose
# kernel code was measured slower and not kept in the tree.)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
if [ -z "$SKIP_TESTS" ]; then
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/fin_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/fin_pytest.log
fi
LIBS=${LIBS:-"paper_1502_02389_b200/liblift.so $(ls build/var_*.so)"}
python scripts/ab.py $LIBS $LIBS 2>&1 | python -c "
import sys,json
for line in sys.stdin:
    line=line.strip()
    if not line.startswith('{\"lib\"'): continue
    a,b=line.split('} ',1); lib=json.loads(a+'}')['lib']
    d=json.loads(b[:b.rindex('}')+1])
    print(lib.ljust(16),' '.join(f'{k}:{v[\"us\"]}' for k,v in d.items()))
"
for l in $LIBS $LIBS; do echo "== $l"; LIFT_LIB=$PWD/$l timeout 300 python scripts/midsize_ab.py; done
for l in $LIBS $LIBS; do echo "== step $l"; LIFT_LIB=$PWD/$l timeout 300 python scripts/step_ab.py 20 2>&1 | python -c "
import sys,json; d=json.load(sys.stdin); print({k:v['ms'] for k,v in d.items() if k in ('seq_events','seq_plain')})"; done
