import sys; sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tests')
import numpy as np
from test_gpu_gemm import _run
for T in [300, 257, 400]:
    for N,K in [(128256,256),(28672,4096)]:
        got, ref = _run(T, N, K, epi=2, seed=T)
        d = np.abs(got-ref); bad = np.argwhere(d > 2e-2*np.abs(ref).max())
        print(T, N, K, "nbad", len(bad), "rows", np.unique(bad[:,0])[:10], "cols", np.unique(bad[:,1]//128)[:20] if len(bad) else "")
