import numpy as np, sys
base = sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/dense_trace'
d=np.loadtxt(base + '.txt',dtype=np.float64)
x=d[d[:,0]==0]; v=x[:,2:6]; t0=v[v>0].min()
n=int((x[:,2]>0).sum()); m=int((x[:,4]>0).sum())
pe=x[:,2]-t0; mf=x[:,4]-t0; mb=x[:,3]-t0
print("producer interval median", np.median(np.diff(pe[:n])), " mma interval median", np.median(np.diff(mf[:m])))
print("mma wait for data median", np.median((mf-mb)[:m]))
tt=x[:,5]; print("MMA tile starts (tempty ready):", (tt[tt>0]-t0)[:8].astype(int))
print("MMA k-block full-ready times at tile boundaries:", mf[[0,15,16,31,32,47,48,63]].astype(int))
e=np.loadtxt(base + '_epi.txt')
for jj in range(4):
    rows=e[e[:,1]==jj]
    st=rows[:,3]-t0; en=rows[:,4]-t0
    ok=rows[:,3]>0
    if ok.any():
        print(f"tile {jj}: epilogue start(tfull) min {st[ok].min():.0f} max {st[ok].max():.0f}; end min {en[ok].min():.0f} max {en[ok].max():.0f}; dur med {np.median((en-st)[ok]):.0f}")
