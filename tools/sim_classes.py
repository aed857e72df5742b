"""Candidates a forward tile scans vs keeps under the support-class binning (CPU replay of
one image per config via the oracle rects; development diagnostic behind DESIGN.md "Binning").
usage: python tools/sim_classes.py"""
import numpy as np, sys
sys.path.insert(0,'/root/repo')
import gsr_synth as S, oracle as O
for (H,W,s) in [(170,255,8.0),(339,510,4.0),(45,68,30.0)]:
    c=S.gaussians(H,W,seed=1000)
    R=O.rects(c,H,W,s,0.1,support=True)   # x0u,y0u,x0,x1,y0,y1 (x1u not given; use clipped+origin)
    ok=(R[:,2]<=R[:,3])&(R[:,4]<=R[:,5]); R=R[ok]
    # unclipped width approx: from sigma: 2*13.5*sigma*s+2
    sg=c["sigma"][ok]
    w=np.ceil(s*13.5*2*sg[:,0])+1; h=np.ceil(s*13.5*2*sg[:,1])+1
    win_w=2*0.1*W*s; win_h=2*0.1*H*s
    w=np.minimum(w,win_w); h=np.minimum(h,win_h)
    TW,TH=32,16
    dens=len(R)/(O.out_dims(H,W,s)[0]*O.out_dims(H,W,s)[1])
    def scanned(cls):
        tot=0
        for k in np.unique(cls):
            m=cls==k
            ew=w[m].max(); eh=h[m].max()
            tot+=m.sum()/len(R)*(ew+TW+15)*(eh+TH+15)*dens
        return tot
    kept=np.mean((w+TW-1)*(h+TH-1))*dens
    m=np.maximum(w,h)
    print((H,W,s),"kept/tile %.0f"%kept,"scan: 1 class %.0f"%scanned(np.zeros(len(m),int)),
          " log2 classes %.0f"%scanned(np.clip(np.floor(np.log2(m))-5,0,3)),
          " sqrt2 classes %.0f"%scanned(np.clip(np.floor(2*np.log2(m))-10,0,7)),
          " 16 cls %.0f"%scanned(np.clip(np.floor(4*np.log2(m))-20,0,15)))
