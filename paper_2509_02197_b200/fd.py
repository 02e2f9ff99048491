"""GPU finite-difference oracle.

Restates the reference's ``finite_difference_gradient`` (verification.py:
53-120): central differences of the dependent with respect to every element
of every independent, all arithmetic in float64 (the program is promoted to
real64 first, verification.py:79-92), per-element step
``sqrt(eps_f64) * max(1, |x|)`` (``fd_epsilon``, :44-50).

Like the reference (``_fd_one``, :95-120) the 2n perturbed copies of an
independent ride the engine's batch axis: they are built on the device and
handed to ``run_forward`` as one leading batch dimension, whose forward
launch list is lowered once and replayed per element (one host
synchronisation per batch). When a data-dependent branch or loop header
differs across the batch (``BatchDivergence``) the elements are probed
pairwise, and a pair that straddles a branch boundary comes back NaN, as in
the reference. The probe batch is cut into chunks of at most
``FD_CHUNK_BYTES`` so memory stays bounded; batch elements are independent,
so chunking does not change any value.
"""
from __future__ import annotations

from dataclasses import replace

import numpy as np

from .ir import Program, adopt


def promote64(program: Program) -> Program:
    """The reference's _promote64 (verification.py:79-92)."""
    if all(d.element_kind == "real64" for d in program.descriptors.values()):
        return program
    return Program(
        descriptors={n: replace(d, element_kind="real64") for n, d in program.descriptors.items()},
        parameters=program.parameters,
        region=program.region,
        dependent=program.dependent,
        independents=program.independents,
    )


FD_CHUNK_BYTES = 256 << 20


def finite_difference_gradient(program, inputs: dict, params: dict | None = None, *, eps: float | None = None,
                               trip_limit=None) -> dict:
    """Central differences on the B200; same arguments and result as the
    reference ``finite_difference_gradient``."""
    import torch

    from .runtime import require_cuda

    require_cuda()
    params = dict(params or {})
    prog = promote64(adopt(program))
    # np.array keeps 0-d inputs 0-d (np.ascontiguousarray would make them 1-d)
    dev = {k: torch.from_numpy(np.array(v, dtype=np.float64, order="C")).cuda() for k, v in inputs.items()}
    return {name: _fd_one(prog, dev, params, name, eps, trip_limit) for name in prog.independents}


def _fd_one(prog, dev, params, name, eps, trip_limit):
    """One independent (reference _fd_one, verification.py:95-120)."""
    import torch

    from .api import run_forward
    from .errors import BatchDivergence

    x = dev[name]
    n = x.numel() if x.dim() else 1
    flat0 = x.reshape(-1)
    if eps is not None:
        h = torch.full_like(flat0, float(eps))
    else:
        h = np.sqrt(np.finfo(np.float64).eps) * torch.clamp(flat0.abs(), min=1.0)

    def probes(lo, hi):
        """Batch of the +h probes of elements [lo, hi) then their -h probes."""
        k = hi - lo
        b = flat0.reshape(1, -1).repeat(2 * k, 1)
        idx = torch.arange(lo, hi, device=x.device)
        rows = torch.arange(k, device=x.device)
        b[rows, idx] += h[lo:hi]
        b[k + rows, idx] -= h[lo:hi]
        return b.reshape((2 * k,) + tuple(x.shape))

    def run(batch):
        r = run_forward(prog, {**dev, name: batch}, params, trip_limit=trip_limit)
        return np.asarray(r.value, dtype=np.float64).reshape(-1)

    hh = h.cpu().numpy()
    g = np.empty(n)
    per = max(1, FD_CHUNK_BYTES // (2 * 8 * max(n, 1)))
    for lo in range(0, n, per):
        hi = min(n, lo + per)
        batch = probes(lo, hi)
        k = hi - lo
        try:
            vals = run(batch)
            g[lo:hi] = (vals[:k] - vals[k:]) / (2.0 * hh[lo:hi])
        except BatchDivergence:
            for i in range(k):
                try:
                    pair = run(batch[[i, k + i]])
                    g[lo + i] = (pair[0] - pair[1]) / (2.0 * hh[lo + i])
                except BatchDivergence:
                    g[lo + i] = np.nan  # the probes straddle a branch boundary
    return g.reshape(tuple(x.shape))
