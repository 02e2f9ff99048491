"""B200-native execution engine for the reverse-mode gradient programs of
gradflow (DaCe AD, arXiv 2509.02197).

Drop-in entry points mirroring the reference:
``gradient``, ``run_planned``, ``run_forward``, ``run_backward`` and
``plan`` (host planner passthrough), and the reference's finite-difference
oracle ``finite_difference_gradient`` on the GPU. Programs arrive as reference objects or
as the reference's JSON wire format (``load_program``/``load_bundle``/
``load_plan``). All data-path work runs as sm_100a kernels from libgfb.so.
"""
from .api import (
    Bundle,
    Engine,
    GradientResult,
    PlanBundle,
    RunResult,
    as_bundle,
    as_plan,
    clear_cache,
    gradient,
    load_bundle,
    load_plan,
    plan,
    plan_from_reference_artifacts,
    run_backward,
    run_forward,
    run_planned,
    save_bundle,
    save_plan,
)
from .errors import *  # noqa: F401,F403
from .fd import finite_difference_gradient
from .ir import Program, adopt, dump_program, load_program

__version__ = "0.1.0"
