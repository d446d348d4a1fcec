cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
LIBS=${LIBS:-"paper_1502_02389_b200/liblift.so build/var_*.so"}
python scripts/ab.py $LIBS 2>&1 | python -c "
import sys,json
for line in sys.stdin:
    line=line.strip()
    if not line.startswith('{\"lib\"'): continue
    a,b=line.split('} ',1); lib=json.loads(a+'}')['lib']
    try: d=json.loads(b.split(' ',0)[0] if False else b[:b.rindex('}')+1])
    except Exception as e: print(lib,'ERR',b[:300]); continue
    print(lib.ljust(14),' '.join(f'{k}:{v[\"us\"]}' for k,v in d.items()))
"
for l in $LIBS; do echo "== step $l"; LIFT_LIB=$PWD/$l timeout 300 python scripts/step_ab.py 20 2>&1 | python -c "
import sys,json; d=json.load(sys.stdin); print({k:v['ms'] for k,v in d.items() if k in ('seq_events','seq_plain','4streams')})"; done
