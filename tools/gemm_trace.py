import ctypes as C, sys
sys.path.insert(0,'/root/repo')
from paper_2501_14784_b200._native import lib, check
for (T,N,K) in [(180,6144,4096),(180,4096,4096),(180,28672,4096),(180,4096,14336),(64,6144,4096),(256,4096,4096)]:
    ms=C.c_float(0); check(lib.ds_dbg_gemm_bench(T,N,K,0,20,0,C.byref(ms))); print("T N K",T,N,K,"us",ms.value*1e3, flush=True)
