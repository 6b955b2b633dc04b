import sys; sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tests')
import numpy as np
from test_gpu_gemm import _run
for (N,K) in [(6144,4096),(4096,4096),(28672,4096),(4096,14336),(128256,4096)]:
    for T in [5,294,318,3]:
        got, ref = _run(T, N, K, epi=2 if N==128256 else 1, seed=T)
        err = np.abs(got-ref).max()/np.abs(ref).max()
        print(N,K,T, "relerr %.4f"%err, "BAD" if err>2e-2 else "")
