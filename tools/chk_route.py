import sys; sys.path.insert(0,'.')
import numpy as np, torch
import paper_2407_14417_b200 as moe
from oracle.oracle import OracleLib
L,E,k,d,f=4,8,2,4096,14336
prof=moe.profile_for_shape(d,f,L,E,k)
plan=moe.make_plan(moe.TaskRequest(moe.QUALITY,0,0),moe.HardwareProfile(10**15),prof)
eng=moe.MoeEngine(L,E,k,d,f,plan,max_tokens=1,seed=0,use_graphs=False)
eng.synth_input(0,1); eng.decode(1); eng.sync()
r=eng.last_routing(1); print('routing',r)
orc=OracleLib(); m=orc.model(L,E,k,d,f,0)
x=orc.step_input(m,0,1)
# gate on layer 0 input with oracle
import ctypes
xd=torch.from_numpy(x.view(np.int16).copy()).cuda()
out=torch.empty(d,dtype=torch.int16,device='cuda'); idx=torch.empty(k,dtype=torch.int32,device='cuda'); w=torch.empty(k,dtype=torch.float32,device='cuda'); lg=torch.empty(E,dtype=torch.float32,device='cuda')
eng.forward_layer(0,xd,1,out,idx,w,lg); eng.sync()
print('gpu idx',idx.cpu().numpy(),'w',w.cpu().numpy(),'lg',lg.cpu().numpy())
ref_out,ref_idx,ref_w,ref_lg=orc.moe_layer(m,0,plan.precision[:E],x.reshape(1,d),1)
print('ref idx',ref_idx,'w',ref_w,'lg',ref_lg)
