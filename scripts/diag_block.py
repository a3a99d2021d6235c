import sys; sys.path.insert(0, "."); sys.path.insert(0, "tests")
import math, time, numpy as np, torch, oracle, sys
sys.path.insert(0,'.'); sys.path.insert(0,'tests')
from paper_2509_19294_b200 import binding, inputs
from test_gpu_block import run_block, eps2_of, _levels_agree
c=inputs.CONFIGS["C1"]; m,x,v=inputs.make("C1")
xg,vg,lg,sg=run_block(m,x,v,c.eps,1/64,4)
xo,vo,_,_,lo,so,co=oracle.hermite_block(m,x,v,eps2_of(c.eps),1/64,4,eta=0.02,eta_s=0.01,kmax=20)
print('C1 traj dx',np.max(np.abs(xg-xo)),'dv',np.max(np.abs(vg-vo)),'lev',_levels_agree(lg,lo,co,1/64),'steps',sg,so, np.bincount(lo))
e2=eps2_of(c.eps); E0=sum(oracle.energy(m,x,v,e2))
xg,vg,_,sg=run_block(m,x,v,c.eps,1/64,16)
xo,vo,*_ ,so2,_=oracle.hermite_block(m,x,v,e2,1/64,16,eta=0.02,eta_s=0.01,kmax=20)
print('C1 drift', abs(sum(oracle.energy(m,xg,vg,e2))-E0)/abs(E0), abs(sum(oracle.energy(m,xo,vo,e2))-E0)/abs(E0), sg)
# C2 block
c=inputs.CONFIGS["C2"]; m,x,v=inputs.make("C2"); e2=eps2_of(c.eps)
t0=time.time(); xg,vg,lg,sg=run_block(m,x,v,c.eps,1/128,1); t1=time.time()
xo,vo,_,_,lo,so,co=oracle.hermite_block(m,x,v,e2,1/128,1,eta=0.02,eta_s=0.01,kmax=20); t2=time.time()
print('C2 1 cycle dt_max=1/128: dx',np.max(np.abs(xg-xo)),'dv',np.max(np.abs(vg-vo)),'lev',_levels_agree(lg,lo,co,1/128),'steps',sg,so,np.bincount(lo),'gpu s',t1-t0,'orc s',t2-t1)
xh,vh,lh,sh=run_block(m,x,v,c.eps,1/128,1,hilo=True)
print('C2 hilo: dx',np.max(np.abs(xh-xo)),'dv',np.max(np.abs(vh-vo)),'lev',_levels_agree(lh,lo,co,1/128),'steps',sh,so,np.bincount(lh), 'plain', np.bincount(lg))
d=np.nonzero(lg!=lo)[0]; print('plain differs at', d[:20], lg[d][:20], lo[d][:20], co[d][:20]*128)
