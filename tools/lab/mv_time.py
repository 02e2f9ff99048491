"""Time the one-pass matrix-vector kernels through the C ABI (fp64 4000^2,
two matrices alternating so the operand is not L2-resident)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2509_02197_b200 import _lib as L

lib = L.load()
R = C = 4000
As = [torch.rand((R, C), device="cuda", dtype=torch.float64) for _ in range(2)]
u = torch.rand(C, device="cuda", dtype=torch.float64)
v = torch.rand(R, device="cuda", dtype=torch.float64)
r = torch.zeros(R, device="cuda", dtype=torch.float64)
c = torch.zeros(C, device="cuda", dtype=torch.float64)
ws = torch.empty(lib.gfb_matvec_pair_workspace_bytes(L.F64, R, C, 1), dtype=torch.uint8, device="cuda")
cs = lambda: torch.cuda.current_stream().cuda_stream
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def t(name, fn, nbytes):
    for i in range(3):
        fn(As[i & 1])
    torch.cuda.synchronize()
    ts = []
    for i in range(20):
        e0.record(); fn(As[i & 1]); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    med = ts[len(ts) // 2]
    # graph replay (how the engine runs): one graph per matrix
    gs = []
    for A in As:
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            fn(A)
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=s):
                fn(A)
        gs.append(g)
    torch.cuda.synchronize()
    tg = []
    for i in range(20):
        e0.record(); gs[i & 1].replay(); e1.record(); e1.synchronize()
        tg.append(e0.elapsed_time(e1))
    tg.sort()
    mg = tg[len(tg) // 2]
    print(f"{name:28s} eager {med*1e3:7.1f} us  {nbytes/med/1e6:7.0f} GB/s   graph {mg*1e3:7.1f} us  {nbytes/mg/1e6:7.0f} GB/s",
          flush=True)


MB = R * C * 8
t("pair chain (atax)", lambda A: lib.gfb_matvec_pair(L.F64, R, C, A.data_ptr(), C, u.data_ptr(), r.data_ptr(), 0, None, c.data_ptr(), 0, 1, ws.data_ptr(), cs()), MB)
t("pair indep (bicg)", lambda A: lib.gfb_matvec_pair(L.F64, R, C, A.data_ptr(), C, u.data_ptr(), r.data_ptr(), 0, v.data_ptr(), c.data_ptr(), 0, 0, ws.data_ptr(), cs()), MB)
t("rows only", lambda A: lib.gfb_matvec_pair(L.F64, R, C, A.data_ptr(), C, u.data_ptr(), r.data_ptr(), 0, None, None, 0, 0, ws.data_ptr(), cs()), MB)
t("cols only", lambda A: lib.gfb_matvec_pair(L.F64, R, C, A.data_ptr(), C, None, None, 0, v.data_ptr(), c.data_ptr(), 0, 0, ws.data_ptr(), cs()), MB)
t("rank2 write", lambda A: lib.gfb_rank2(L.F64, R, C, v.data_ptr(), u.data_ptr(), v.data_ptr(), u.data_ptr(), A.data_ptr(), C, 0, cs()), MB)
t("rank2 accumulate", lambda A: lib.gfb_rank2(L.F64, R, C, v.data_ptr(), u.data_ptr(), v.data_ptr(), u.data_ptr(), A.data_ptr(), C, 1, cs()), 2 * MB)
t("rank1 write", lambda A: lib.gfb_rank2(L.F64, R, C, v.data_ptr(), u.data_ptr(), None, None, A.data_ptr(), C, 0, cs()), MB)
t("torch copy (r+w)", lambda A: As[0 if A is As[1] else 1].copy_(A), 2 * MB)
