"""One gfb_matmul fp32 call of a chosen mlp shape (for ncu): python mm_one.py M N K ta tb"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2509_02197_b200 import _lib as L

M, N, K, ta, tb = (int(x) for x in sys.argv[1:6])
lib = L.load()
A = torch.rand((K, M) if ta else (M, K), device="cuda") + 0.1
B = torch.rand((N, K) if tb else (K, N), device="cuda") + 0.1
C = torch.empty((M, N), device="cuda")
ws = torch.empty(max(lib.gfb_matmul_workspace_bytes(L.F32, ta, tb, M, N, K), 16), dtype=torch.uint8, device="cuda")
for _ in range(3):
    L.check(lib.gfb_matmul(L.F32, ta, tb, M, N, K, A.data_ptr(), A.shape[1], B.data_ptr(), B.shape[1], C.data_ptr(), N,
                           0, ws.data_ptr(), torch.cuda.current_stream().cuda_stream), "matmul")
torch.cuda.synchronize()
print("ok")
