import numpy as np, sys
d=np.loadtxt(sys.argv[1] if len(sys.argv)>1 else 'gpurun_out/dense_trace.txt',dtype=np.float64)
for b in (0,1):
    x=d[d[:,0]==b]; v=x[:,2:5]; t0=v[v>0].min()
    pe=x[:,2]-t0; mb=x[:,3]-t0; mf=x[:,4]-t0
    n=int((x[:,2]>0).sum())
    print("block",b,"kblocks traced",n)
    print(" producer empty-ready:", pe[:12].astype(int))
    dp=np.diff(pe[:n]); print(" producer interval median", np.median(dp), "mean", dp.mean())
    if b==0:
        m=int((x[:,4]>0).sum())
        print(" mma full-ready:", mf[:12].astype(int))
        dk=np.diff(mf[:m]); print(" mma per-kblock interval: median", np.median(dk), "mean", dk.mean())
        print(" mma wait for data median:", np.median((mf-mb)[:m]))
        tt=x[:,5]; print(" tile starts:", (tt[tt>0]-t0)[:8].astype(int))
