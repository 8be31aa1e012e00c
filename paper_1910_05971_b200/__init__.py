"""B200-native FastSV connected components (arXiv 1910.05971).

A drop-in for the reference package ``svcc``'s hot path
(``fastsv_la``/``fastsv``, /root/reference/pkg/src/svcc/driver.py:64-120):
the same Python entry points and result types, with every iteration run by
hand-written sm_100a kernels behind the C ABI of ``include/fastsv.h``.
"""

from .driver import (DriverConfig, HookingConfig, IterationTrace, RunResult, Solver,
                     ablation_results, ablation_suite, choose_kernel, connected_components,
                     default_solver, device_count, fastsv, fastsv_la, require_device,
                     simplified_sv, sv_level_config)
from .errors import DeviceError, InputError, InvariantError, SvccError, VerificationError
from ._native import FsvStats
from .graph import ComponentSizes, CsrGraph, Labeling, build_csr, labeling_from_parents

__version__ = "0.1.0"

__all__ = [
    "CsrGraph", "Labeling", "ComponentSizes", "build_csr", "labeling_from_parents", "FsvStats",
    "DriverConfig", "HookingConfig", "IterationTrace", "RunResult", "Solver",
    "choose_kernel", "fastsv_la", "fastsv", "connected_components", "default_solver",
    "simplified_sv", "sv_level_config", "ablation_results", "ablation_suite",
    "device_count", "require_device",
    "SvccError", "InputError", "VerificationError", "InvariantError", "DeviceError",
    "__version__",
]
