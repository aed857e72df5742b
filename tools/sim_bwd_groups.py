"""Replays the backward grouping on the binning of one C5 image (CPU, via the oracle rects):
fraction of evaluated lane-pairs that fall inside the lane's own support rect, for several group
orderings and tile shapes (development diagnostic behind DESIGN.md "K5 backward").
usage: python tools/sim_bwd_groups.py"""
import numpy as np, sys
sys.path.insert(0,'/root/repo')
import gsr_synth as S, oracle as O
H,W,s=170,255,8.0
c=S.gaussians(H,W,seed=1000)
R=O.rects(c,H,W,s,0.1,support=True)
ok=(R[:,2]<=R[:,3])&(R[:,4]<=R[:,5]); R=R[ok]
Hs,Ws=O.out_dims(H,W,s)
offx=16*((int(np.ceil(2*s*0.1*W))+2+15)//16); offy=16*((int(np.ceil(2*s*0.1*H))+2+15)//16)
cx=(R[:,0]+offx)//16; cy=(R[:,1]+offy)//16; ncx=(Ws+offx+15)//16
order=np.argsort(cy*ncx+cx,kind='stable'); R=R[order]
def run(TW,TH,mode):
    U=Wk=0
    for Tx0 in range(640,1400,TW):
        for Ty0 in range(320,1000,TH):
            Tx1=Tx0+TW-1; Ty1=Ty0+TH-1
            hit=~((R[:,3]<Tx0)|(R[:,2]>Tx1)|(R[:,5]<Ty0)|(R[:,4]>Ty1))
            idx=np.nonzero(hit)[0]
            x0=np.maximum(R[idx,2],Tx0); x1=np.minimum(R[idx,3],Tx1); y0=np.maximum(R[idx,4],Ty0); y1=np.minimum(R[idx,5],Ty1)
            U+=((x1-x0+1)*(y1-y0+1)).sum()
            if mode=='x0': o=np.argsort(x0,kind='stable')
            elif mode=='x0x1': o=np.lexsort((x1,x0))
            elif mode=='y0x0': o=np.lexsort((x0,y0))
            elif mode=='cls': o=np.lexsort((x0, (x0>Tx0).astype(int)*2+(x1<Tx1).astype(int), (y0>Ty0).astype(int)*2+(y1<Ty1).astype(int)))
            else: o=np.arange(len(idx))
            x0,x1,y0,y1=x0[o],x1[o],y0[o],y1[o]
            for g in range(0,len(idx),32):
                sl=slice(g,g+32)
                Wk+=32*(x1[sl].max()-x0[sl].min()+1)*(y1[sl].max()-y0[sl].min()+1)
    return U/Wk
for TW,TH in [(64,32),(32,32)]:
    print(TW,TH,{m:round(run(TW,TH,m),3) for m in ['none','x0','x0x1','y0x0','cls']})
def run2(TW,TH,q,batch=None,withy=False):
    U=Wk=0
    for Tx0 in range(640,1400,TW):
        for Ty0 in range(320,1000,TH):
            Tx1=Tx0+TW-1; Ty1=Ty0+TH-1
            hit=~((R[:,3]<Tx0)|(R[:,2]>Tx1)|(R[:,5]<Ty0)|(R[:,4]>Ty1))
            idx=np.nonzero(hit)[0]
            x0=np.maximum(R[idx,2],Tx0)-Tx0; x1=np.minimum(R[idx,3],Tx1)-Tx0; y0=np.maximum(R[idx,4],Ty0)-Ty0; y1=np.minimum(R[idx,5],Ty1)-Ty0
            U+=((x1-x0+1)*(y1-y0+1)).sum()
            n=len(idx); B=batch or n
            for b0 in range(0,n,B):
                sl=slice(b0,b0+B)
                k=(x0[sl]>>q)*64+(x1[sl]>>q)
                if withy: k=k*64+(y0[sl]>>q)*8+(y1[sl]>>q)
                o=np.argsort(k,kind='stable')
                a0,a1,c0,c1=x0[sl][o],x1[sl][o],y0[sl][o],y1[sl][o]
                for g in range(0,len(o),32):
                    s2=slice(g,g+32)
                    Wk+=32*(a1[s2].max()-a0[s2].min()+1)*(c1[s2].max()-c0[s2].min()+1)
    return U/Wk
for q in [2,3,4]:
    print("64x32 bucket q",q, round(run2(64,32,q),3), "batch1024", round(run2(64,32,q,1024),3), "batch512", round(run2(64,32,q,512),3), "withy", round(run2(64,32,q,1024,True),3))
