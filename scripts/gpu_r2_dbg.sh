cd "${GRAFT_REPO_ROOT:-/root/repo}"
LIFT_LIB=$PWD/build/tune/load_tma_bulk.so python - <<'PY' 2>&1 | tail -5
import torch, lift_inputs as gen, paper_1502_02389_b200 as lift
dev=torch.device("cuda:0")
for n in (1, 9, 8191, 8192*3+5, 1<<20):
    x=gen.fill_device(torch.empty(n,device=dev),1,1,0,0,-1.,1.); y=gen.fill_device(torch.empty(n,device=dev),1,2,0,0,-1.,1.)
    for name,f in (("scal",lambda: lift.scal(3.0,x)),("asum",lambda: lift.asum(x)),("dot",lambda: lift.dot(x,y))):
        try: f(); torch.cuda.synchronize(); print(n,name,"ok")
        except Exception as e: print(n,name,"FAIL",e)
PY
