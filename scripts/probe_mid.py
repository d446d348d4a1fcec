import sys, torch; sys.path.insert(0,'.')
import lift_inputs as gen, paper_1502_02389_b200 as lift
x=gen.fill_device(torch.empty(1<<24,device='cuda'),0,1,0,0,-1.0,1.0)
ws=lift.Workspace(1<<24, torch.device('cuda'))
r=torch.empty(1,device='cuda')
for _ in range(3): lift.asum(x,out=r,ws=ws)
torch.cuda.synchronize()
