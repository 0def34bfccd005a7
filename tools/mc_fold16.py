"""Monte Carlo of the fast-path filters on random g-subsets of a config's Gamma_j (CPU, host prep only):
the 32-bit probe fold, its 16-bit fold and the pair-sum test of two 16-bit folds in one POPC.
Usage: PYTHONPATH=. python tools/mc_fold16.py <config> <g> <thr0>"""
import paper_2408_10743_b200 as P, numpy as np, sys
cid=int(sys.argv[1]) if len(sys.argv)>1 else 4
g=int(sys.argv[2]) if len(sys.argv)>2 else 9
thr=int(sys.argv[3]) if len(sys.argv)>3 else 9
c=P.CONFIGS[cid]; a=P.generate_code(c['n'],c['k'],c['seed']); n=c['n']
gs=P.information_sets(P.isometry_transform(a))
rng=np.random.default_rng(1)
W=(n+31)//32
for j,gm in enumerate(gs):
    M=np.asarray(gm.matrix,dtype=np.uint8)  # rows x 3n
    N=M.shape[0]
    x=M[:,:n]; z=M[:,n:2*n]
    # pack into W 32-bit words per half
    def pack(h):
        pad=np.zeros((N,W*32),dtype=np.uint8); pad[:,:n]=h
        return np.packbits(pad.reshape(N,W,32),axis=2,bitorder='little').view('<u4').reshape(N,W)
    X=pack(x); Z=pack(z)
    # orientation per block: denser component as probe (sample 6-row sums)
    S=rng.integers(0,N,size=(512,6))
    probe=np.zeros((N,W),dtype=np.uint32)
    for w in range(W):
        sx=np.bitwise_xor.reduce(X[S,w],axis=1); sz=np.bitwise_xor.reduce(Z[S,w],axis=1)
        dx=np.unpackbits(sx.view(np.uint8)).sum(); dz=np.unpackbits(sz.view(np.uint8)).sum()
        probe[:,w]= X[:,w] if dx>=dz else Z[:,w]
    # random g-subsets: fold32 = OR_w probe sums
    T=400000
    idx=np.argsort(rng.random((T,N)),axis=1)[:,:g]
    sums=np.bitwise_xor.reduce(probe[idx],axis=1)  # T x W
    u=np.bitwise_or.reduce(sums,axis=1).astype(np.uint32)
    pc32=np.unpackbits(u.view(np.uint8).reshape(-1,4),axis=1).sum(1)
    f16=(u|(u>>16))&0xFFFF
    pc16=np.unpackbits(f16.astype(np.uint16).view(np.uint8).reshape(-1,2),axis=1).sum(1)
    s=pc16[0::2]+pc16[1::2]
    print(f"gamma {j}: N={N} mean popc32 {pc32.mean():.2f} P(pc32<={thr}) {np.mean(pc32<=thr):.2e}  mean N16 {pc16.mean():.2f} P(N16<={thr}) {np.mean(pc16<=thr):.2e}  P(pair s<={thr+16}) {np.mean(s<=thr+16):.2e}")
