"""GPU finite-difference oracle.

Restates the reference's ``finite_difference_gradient`` (verification.py:
53-120): central differences of the dependent with respect to every element
of every independent, all arithmetic in float64 (the program is promoted to
real64 first, verification.py:79-92), per-element step
``sqrt(eps_f64) * max(1, |x|)`` (``fd_epsilon``, :44-50).

The reference rides its interpreter's batch axis (2n perturbed copies in one
run). Here the promoted forward program is lowered once into a device launch
list that is replayed as a CUDA graph: per probe, one element of the
independent is perturbed in HBM, the list runs, and the dependent is copied
into a device vector; there is a single host synchronisation per
independent. Programs with data-dependent branches are not lowered
(UnsupportedConstruct), so the reference's pairwise BatchDivergence fallback
has no counterpart.
"""
from __future__ import annotations

from dataclasses import replace

import numpy as np

from .errors import UnboundName
from .ir import Program, adopt, number_writes


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


def finite_difference_gradient(program, inputs: dict, params: dict | None = None, *, eps: float | None = None,
                               trip_limit=None) -> dict:
    """Central differences on the B200; same arguments and result as the
    reference ``finite_difference_gradient``."""
    import torch

    from .api import _check_inputs, _init_env
    from .lowering import Lowering, ProgramRun
    from .runtime import Executable, require_cuda

    require_cuda()
    params = dict(params or {})
    prog = promote64(adopt(program))
    base = {k: np.asarray(v, dtype=np.float64) for k, v in inputs.items()}
    shapes = _check_inputs(prog, base, params)
    low = Lowering(trip_limit=trip_limit)
    env, ins = _init_env(low, prog, shapes, "")
    ProgramRun(low, prog, params, env, versions=number_writes(prog)).run()
    dep = env.get(prog.dependent)
    if dep is None:
        raise UnboundName(f"dependent '{prog.dependent}' was never written")
    low.finish([dep])
    exe = Executable(low, ins, {"value": low.resolve(dep)})
    dev = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in base.items()}
    value = exe.output("value")
    grads = {}
    for name in prog.independents:
        x0 = dev[name]
        n = x0.numel() if x0.dim() else 1
        h = np.sqrt(np.finfo(np.float64).eps) * torch.clamp(x0.reshape(-1).abs(), min=1.0)
        if eps is not None:
            h = torch.full_like(h, float(eps))
        probe = x0.clone()
        flat = probe.reshape(-1)
        vals = torch.empty(2 * n, dtype=torch.float64, device=x0.device)
        run_inputs = dict(dev)
        run_inputs[name] = probe
        errs = torch.zeros_like(exe.err)
        for i in range(n):
            for s, j in ((1.0, i), (-1.0, n + i)):
                flat[i] = x0.reshape(-1)[i] + s * h[i]
                exe.run(run_inputs, sync=False)
                vals[j] = value.reshape(())
                errs.bitwise_or_(exe.err)
            flat[i] = x0.reshape(-1)[i]
        # one synchronisation per independent: domain errors of any probe
        # propagate (a gradient at an invalid point is not defined)
        bits = int(errs.item())
        if bits:
            from . import _lib as L
            from .errors import DomainError

            raise DomainError("; ".join(m for b, m in L.EBITS.items() if bits & b) or f"device error bits {bits:#x}")
        g = (vals[:n] - vals[n:]) / (2.0 * h)
        grads[name] = g.reshape(x0.shape).cpu().numpy()
    return grads
