import sys, numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "oracle")
import paper_2605_19388_b200 as dfm, oracle
for (F,T) in [(5,300),(9,57),(33,400)]:
    sizes=[4]*8; N=8; K=32
    layout=dfm.BlockLayout(sizes)
    x=dfm.generate_mixture(1,F,T,32,N,K,4); init=dfm.random_init(F,T,layout,N,K,8)
    fit=dfm.fit_distributed(x,layout,init,6,True)
    ref=oracle.run_engine(x,sizes,dict(T=init.nmf.T,V=init.nmf.V,lam=init.lambda0,w=init.w0),6)
    print(F,T,np.max(np.abs(fit.report.cost_trace-ref['cost_trace'])/np.abs(ref['cost_trace'])), flush=True)
