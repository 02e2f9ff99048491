"""Dump gfb_matmul fp32 results of the mlp shapes (fixed seed) to an npz, to
compare libraries bit for bit: python mm_bits.py out.npz"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
from paper_2509_02197_b200 import _lib as L
from mm_time import SHAPES  # noqa: E402

lib = L.load()
out = {}
g = torch.Generator(device="cuda").manual_seed(0)
for i, (M, N, K, ta, tb, lab) in enumerate(SHAPES):
    A = torch.randn((K, M) if ta else (M, K), device="cuda", generator=g)
    B = torch.randn((N, K) if tb else (K, N), device="cuda", generator=g)
    C = torch.empty((M, N), device="cuda")
    ws = torch.empty(max(lib.gfb_matmul_workspace_bytes(L.F32, ta, tb, M, N, K), 16), dtype=torch.uint8, device="cuda")
    L.check(lib.gfb_matmul(L.F32, ta, tb, M, N, K, A.data_ptr(), A.shape[1], B.data_ptr(), B.shape[1], C.data_ptr(), N,
                           0, ws.data_ptr(), torch.cuda.current_stream().cuda_stream), "matmul")
    ref = (A.double().T if ta else A.double()) @ (B.double().T if tb else B.double())
    err = ((C.double() - ref).abs() / ref.abs().clamp(min=1)).max().item()
    print(f"{lab:16s} err {err:.2e}")
    out[f"c{i}"] = C.cpu().numpy()
np.savez(sys.argv[1], **out)
if len(sys.argv) > 2:
    ref = np.load(sys.argv[2])
    for k in out:
        d = np.count_nonzero(out[k].view(np.uint32) != ref[k].view(np.uint32))
        print(k, "differing elements:", d, "of", out[k].size)
