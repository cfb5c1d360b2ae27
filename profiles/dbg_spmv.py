import sys, os; sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tests')
import numpy as np, torch, oracle as O, workloads as W
import paper_2604_17198_b200 as N
from util import random_csr
def dev(A): return W.SparseMatrix(A.format,A.nrows,A.ncols,*(torch.from_numpy(t).cuda() if t is not None else None for t in (A.pos,A.crd,A.val,A.outer_crd)))
for dtype in (np.float32, np.float64):
  rng=np.random.default_rng(11)
  for trial in range(15):
    M,Nc=int(rng.integers(1,5000)),int(rng.integers(1,3000))
    A=random_csr(rng,M,Nc,float(rng.uniform(0.0005,0.01)),dtype=dtype,dense_rows=[int(rng.integers(M))] if trial%2==0 else (),empty_frac=0.4)
    x=rng.uniform(0.5,1.5,Nc).astype(dtype)
    Ad,xd=dev(A),torch.from_numpy(x).cuda()
    ref=O.spmv(A,x)
    for P in (None,1,3,64,A.nnz+5):
      for rep in range(3):
        parts=N.partition([Ad],P) if P else None
        y=N.spmv(Ad,xd,parts).cpu().numpy()
        bad=np.nonzero(~np.isclose(y,ref,rtol=1e-5))[0]
        if len(bad):
            r=bad[0]
            print(dtype.__name__,"trial",trial,"rep",rep,"P",P,"M",M,"nnz",A.nnz,"bad rows",bad[:5],"y",y[bad[:3]],"ref",ref[bad[:3]],"rowlen",A.pos[r+1]-A.pos[r], "pos", A.pos[r], A.pos[r+1], "first nonempty", np.nonzero(np.diff(A.pos))[0][:3])
