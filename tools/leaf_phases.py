"""Leaf-phase profile of k_base_big (build with tools/build_var.sh ph -DPDQ_BIG_PHASES, run with
PDQ_LIB=tools/libvar_ph.so): share of thread-0 cycles per phase and cycles per leaf."""
import sys
sys.path.insert(0,'/root/repo')
import torch
from paper_2106_05123_b200 import DeviceSorter
n=1<<28
g=torch.Generator(device='cuda'); g.manual_seed(1)
src=torch.randint(-(2**31),2**31,(n,),device='cuda',generator=g,dtype=torch.int64).to(torch.int32)
ds=DeviceSorter(n,torch.int32,False)
for r in range(3):
    x=src.clone(); ds.run(x); st=ds.finish()
tot=st['sched_retire']+st['sched_claim']+st['sched_fetch']+st['sched_idle']
print({k:round(st[k]/tot,3) for k in ['sched_retire','sched_claim','sched_fetch','sched_idle']}, 'cycles per leaf', tot/st['base_cases'])
