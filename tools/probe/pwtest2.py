import numpy as np, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import oracle as O, paper_1911_10175_b200 as sp
V=16
n,C,K,H,W,st = 16,256,64,56,56,1
sh=sp.ConvShape.make(n,C,K,H,W,1,1,st,st)
D=O.gen_sparse(n,C,H,W,0.5,1); dY=O.gen_sparse(n,K,sh.out_h(),sh.out_w(),0.0,2)
ref=O.dense(2,sh.astuple(),D,dY)
pl=sp.plan(sh,sp.Component.bww,V)
a,b=sp.pack_act_chwnn(D,V).to("cuda"),sp.pack_act_nchwc(dY,V).to("cuda")
outs=[]
for rep in range(4):
    res=sp.run_parallel(a,b,sh,pl,sp.RunMode.sparse)
    got=sp.unpack(res.out).cpu().numpy(); outs.append(got)
    d=np.abs(got-ref)/np.abs(ref).max()
    bad=np.argwhere(d>1e-5)
    print(rep,'err',d.max(),'nbad',len(bad),'same as first',np.array_equal(got,outs[0]), 'bad k',sorted(set(bad[:,0].tolist()))[:8],'bad c',sorted(set(bad[:,1].tolist()))[:16], 'rel of bad', (got-ref)[tuple(bad[0])]/ref[tuple(bad[0])] if len(bad) else None)
