"""Time gfb_matmul fp32 on the mlp shapes (graph replay) against cuBLAS fp32
(torch.matmul with TF32 off) and the HBM floor of the shape."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2509_02197_b200 import _lib as L

torch.backends.cuda.matmul.allow_tf32 = False
lib = L.load()
cs = lambda: torch.cuda.current_stream().cuda_stream
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
SHAPES = [  # (M, N, K, ta, tb, label)
    (64, 4096, 512, 0, 0, "fwd x@W1"), (64, 4096, 4096, 0, 0, "fwd r1@W2"), (64, 1024, 4096, 0, 0, "fwd r2@W3"),
    (64, 4096, 1024, 0, 1, "bwd z3g@W3^T"), (4096, 1024, 64, 1, 0, "bwd r2^T@z3g"),
    (64, 4096, 4096, 0, 1, "bwd z2g@W2^T"), (4096, 4096, 64, 1, 0, "bwd r1^T@z2g"),
    (64, 512, 4096, 0, 1, "bwd z1g@W1^T"), (512, 4096, 64, 1, 0, "bwd x^T@z1g"),
]


def timeit(fn):
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn(); torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(30):
        e0.record(); g.replay(); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2] * 1e3


def main():
    tot_ours = tot_cub = 0
    for M, N, K, ta, tb, lab in SHAPES:
        A = torch.rand((K, M) if ta else (M, K), device="cuda") + 0.1
        B = torch.rand((N, K) if tb else (K, N), device="cuda") + 0.1
        C = torch.empty((M, N), device="cuda")
        ws = torch.empty(max(lib.gfb_matmul_workspace_bytes(L.F32, ta, tb, M, N, K), 16), dtype=torch.uint8, device="cuda")
        f = lambda: lib.gfb_matmul(L.F32, ta, tb, M, N, K, A.data_ptr(), A.shape[1], B.data_ptr(), B.shape[1], C.data_ptr(), N, 0, ws.data_ptr(), cs())
        ours = timeit(f)
        ref = (A.double().T if ta else A.double()) @ (B.double().T if tb else B.double())
        err = ((C.double() - ref).abs() / ref.abs().clamp(min=1)).max().item()
        opA = A.T if ta else A
        opB = B.T if tb else B
        cub = timeit(lambda: torch.matmul(opA, opB, out=C))
        byts = 4 * (M * K + K * N + M * N)
        tot_ours += ours; tot_cub += cub
        print(f"{lab:16s} M={M:5d} N={N:5d} K={K:5d}  ours {ours:7.1f} us ({byts/ours/1e3:6.0f} GB/s, {2*M*N*K/ours/1e6:6.1f} TF/s) err {err:.1e}   cublas-fp32 {cub:7.1f} us", flush=True)
    print(f"total ours {tot_ours:.1f} us, cublas fp32 {tot_cub:.1f} us")


if __name__ == "__main__":
    main()
