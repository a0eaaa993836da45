"""paper_1906_04572_b200 — B200-native (sm_100a) CoR-UTV and ALM-CoRUTV.

Drop-in for the hot path of the reference package ``corutv``
(/root/reference/pkg/src/corutv): ``corutv(a, cfg, counter=None)`` and
``alm_corutv(m, cfg)`` with the same configs, result types and exceptions,
computed by hand-written CUDA kernels (libcorutv_b200.so, C-ABI in
include/corutv_b200.h).  There is no CPU fallback.

:func:`install` rebinds the reference package's names to this
implementation: ``corutv.sketch.corutv``, ``corutv.rpca.corutv``,
``corutv.bench.corutv``, ``corutv.corutv``, ``corutv.rpca.alm_corutv``,
``corutv.alm_corutv``, ``sor_svd`` / ``tsr_svd`` and the InexactALM baseline
(``corutv.rpca.inexact_alm``, ``corutv.rpca.svt``).
"""

from .dense import frobenius_norm, singular_values, spectral_norm
from .errors import ConvergenceError, CorutvError
from .rpca import (AlmConfig, RpcaSolution, alm_corutv, corutv_threshold, inexact_alm, shrink, svt,
                   write_telemetry_csv)
from .sketch import (
    VARIANT_APPROX,
    VARIANT_EXACT,
    CorUtvFactors,
    PassCounter,
    SketchConfig,
    corutv,
    corutv_kpq,
    corutv_lowrank_error,
    count_passes,
    flop_estimate,
    gaussian_matrix,
    sor_svd,
    tsr_svd,
)
from .dense import SvdFactors, jacobi_svd

__version__ = "0.1.0"

__all__ = [
    "AlmConfig", "ConvergenceError", "CorUtvFactors", "CorutvError", "PassCounter",
    "RpcaSolution", "SketchConfig", "VARIANT_APPROX", "VARIANT_EXACT", "alm_corutv", "corutv",
    "corutv_kpq", "corutv_lowrank_error", "corutv_threshold", "count_passes", "flop_estimate",
    "frobenius_norm", "gaussian_matrix", "install", "shrink", "singular_values", "spectral_norm",
    "write_telemetry_csv", "sor_svd", "tsr_svd", "SvdFactors", "inexact_alm", "svt", "jacobi_svd",
]


def install(ref_pkg=None):
    """Rebind the reference package's hot-path entry points to the device
    implementation (the binding a maintainer adds).
    Returns the list of rebound ``module.name`` strings."""
    import importlib

    if ref_pkg is None:
        ref_pkg = importlib.import_module("corutv")
    done = []
    for modname, name, obj in (
        ("sketch", "corutv", corutv),
        ("sketch", "sor_svd", sor_svd),
        ("sketch", "tsr_svd", tsr_svd),
        ("rpca", "corutv", corutv),
        ("bench", "corutv", corutv),
        ("rpca", "alm_corutv", alm_corutv),
        ("bench", "alm_corutv", alm_corutv),
        ("rpca", "inexact_alm", inexact_alm),
        ("bench", "inexact_alm", inexact_alm),
        ("rpca", "svt", svt),
    ):
        try:
            mod = importlib.import_module(f"{ref_pkg.__name__}.{modname}")
        except ImportError:
            continue
        if hasattr(mod, name):
            setattr(mod, name, obj)
            done.append(f"{mod.__name__}.{name}")
    for name, obj in (("corutv", corutv), ("alm_corutv", alm_corutv)):
        setattr(ref_pkg, name, obj)
        done.append(f"{ref_pkg.__name__}.{name}")
    for name, obj in (("sor_svd", sor_svd), ("tsr_svd", tsr_svd), ("inexact_alm", inexact_alm), ("svt", svt)):
        if hasattr(ref_pkg, name):
            setattr(ref_pkg, name, obj)
            done.append(f"{ref_pkg.__name__}.{name}")
    return done
