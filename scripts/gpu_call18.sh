#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -k blackscholes > gpurun_out/pytest_bs.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_bs.log
tail -15 gpurun_out/pytest_bs.log
timeout 600 python scripts/ab.py build/liblift_cur.so > gpurun_out/ab18.log 2>&1
cat gpurun_out/ab18.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"blackscholes" -s 1 -c 1 -o gpurun_out/r1_bs python -c "
import torch, sys; sys.path.insert(0,'.')
import lift_inputs as gen, paper_1502_02389_b200 as lift
s=gen.fill_device(torch.empty(4<<20,device='cuda'),0,1,0,0,10.0,200.0)
for _ in range(3): lift.blackscholes(s,100.0,0.05,0.2,1.0)
torch.cuda.synchronize()" > gpurun_out/r1_bs_ncu.log 2>&1
echo "ncu rc=$?"
