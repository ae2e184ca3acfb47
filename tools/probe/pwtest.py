import numpy as np, sys
sys.path.insert(0,'/root/repo')
import oracle as O, paper_1911_10175_b200 as sp
V=16
for (n,C,K,H,W,st) in [(16,256,64,56,56,1),(16,256,64,28,28,1),(16,256,64,14,14,1),(16,256,64,16,16,1),(16,128,64,56,56,1),(16,64,64,6,6,1),(16,64,128,6,6,1),(16,128,64,6,6,1),(16,128,128,6,6,1),(16,256,64,6,6,1),(16,256,128,5,7,1),(20,128,256,6,6,2),(3,256,64,4,4,1)]:
    sh=sp.ConvShape.make(n,C,K,H,W,1,1,st,st)
    D=O.gen_sparse(n,C,H,W,0.5,1); dY=O.gen_sparse(n,K,sh.out_h(),sh.out_w(),0.0,2)
    ref=O.dense(2,sh.astuple(),D,dY)
    pl=sp.plan(sh,sp.Component.bww,V)
    res=sp.run_parallel(sp.pack_act_chwnn(D,V).to("cuda"),sp.pack_act_nchwc(dY,V).to("cuda"),sh,pl,sp.RunMode.sparse)
    got=sp.unpack(res.out).cpu().numpy()
    err=O.max_abs_rel(got,ref)
    bad=np.argwhere(np.abs(got-ref)>1e-3*np.abs(ref).max())
    print((n,C,K,H,W,st),'err',err,'nbad',len(bad), 'first bad (k,c,..)', bad[:4].tolist(), 'bad k set', sorted(set(bad[:,0].tolist()))[:10], 'bad c set', sorted(set(bad[:,1].tolist()))[:12])
