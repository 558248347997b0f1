"""Step-parallel tail estimate (profiling helper): per-pixel sample counts of the REFERENCE render
(oracle/_ref) of ring view 3, grouped as K5 compacts hit rays into warps; compares lane-parallel
warp iterations with a hybrid that switches a warp to step-parallel marching (cost factor 2.5 per
32-step chunk) once at most A lanes are live. Usage: python tools/sim_tail.py K M W"""
import sys, numpy as np
sys.path.insert(0,'/root/repo')
from oracle.bindings import RefCore, RefScene, ref_shell_camera
ref=RefCore(); K,M,W=[int(x) for x in sys.argv[1:4]]
sc=RefScene(ref,K,M)
k9,r9,t3=ref_shell_camera(ref,3,64,W)
tot,rgb,a,S=sc.render(k9,r9,t3,W,W,outputs=True)
S=S.reshape(W,W)
np.save(f'/tmp/S_{K}_{M}_{W}.npy', S)
tid=np.arange(128); wid,lane=tid>>5,tid&31
for NT in (128,):
  lx=(wid&1)*8+(lane&7); ly=(wid>>1)*4+(lane>>3)
  base=0; lanepar=0; work=0
  res={A:0.0 for A in (0,4,8,12,16)}
  for ty in range(W//16):
    for half in range(2):
      for tx in range(W//16):
        v=S[ty*16+half*8+ly, tx*16+lx]; h=v[v>0]
        for i in range(0,len(h),32):
          g=np.sort(h[i:i+32])[::-1]; work+=g.sum(); lanepar+=g.max()
          for A in res:
            # run lane-parallel until active lanes <= A, then step-parallel for remaining with cost factor 2.5 per 32 steps
            if A==0: res[A]+=g.max(); continue
            n=len(g)
            if n<=A: t_switch=0
            else: t_switch=g[A]  # the (A+1)-th longest ray ends at g[A]: after that <=A active
            rem=np.clip(g[:A]-t_switch,0,None)
            res[A]+=t_switch+2.5*np.ceil(rem/32).sum()
  print(f'K={K} work/lanepar (within-warp eff) {work/(32*lanepar):.3f}')
  for A,v in res.items(): print(f'  tail threshold {A}: warp-iterations {v/lanepar:.3f} of lane-parallel')
