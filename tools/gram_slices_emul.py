import numpy as np
rng=np.random.default_rng(0)
n,s=4000,48
# RFF-like features: sqrt(2/s) cos
z=np.sqrt(2/512)*np.cos(rng.standard_normal((n,s))*3+rng.uniform(0,2*np.pi,s))
zl=z.astype(np.longdouble)
Gex=(zl.T@zl)
G64=z.T@z
def old(z):
    m=np.abs(z).max(0); e=np.floor(np.log2(m)).astype(int)+1
    w=np.ldexp(z,7-e[None,:])
    digs=[]
    for p in range(8):
        a=np.trunc(w); digs.append(a.astype(np.int64)); w=(w-a)*128.0
    G=np.zeros((s,s),dtype=np.longdouble)
    gc=[sum(digs[p].T@digs[c-p] for p in range(c+1)) for c in range(8)]
    acc=sum(gc[c].astype(np.longdouble)*np.longdouble(2.0)**(-7*c) for c in range(8))
    return acc*np.exp2((e[:,None]+e[None,:]-14).astype(np.longdouble))
def new(z):
    m=np.abs(z).max(0); e=np.floor(np.log2(m)).astype(int)+2
    e+= (np.ldexp(m,-e)>0.498)
    U=np.rint(np.ldexp(z,56-e[None,:])).astype(np.int64)
    digs=[None]*7
    for p in range(6,-1,-1):
        d=((U&0xFF)^0x80)-0x80
        digs[p]=d; U=(U-d)>>8
    gc=[sum(digs[p].T@digs[c-p] for p in range(c+1)) for c in range(7)]
    H=(gc[0]*256+gc[1])*256+gc[2]
    Lo=((gc[3]*256+gc[4])*256+gc[5])*256+gc[6]
    val=H.astype(np.float64)+Lo.astype(np.float64)*2.0**-32   # kernel: fma(double(Lo),2^-32,double(H))
    return np.ldexp(val,(e[:,None]+e[None,:]-32))
for name,G in (("fp64 dot",G64),("old 36",old(z)),("new 28",new(z))):
    err=np.abs(G.astype(np.longdouble)-Gex)
    print(name, "max abs err", float(err.max()), "max rel-to-diag", float((err/np.sqrt(np.outer(np.diag(Gex),np.diag(Gex)))).max()), "rms", float(np.sqrt((err**2).mean())))
