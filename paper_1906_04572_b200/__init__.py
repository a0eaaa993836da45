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


def _adopt_reference_errors(errs) -> bool:
    """Make the exceptions this package raises also instances of the
    reference's own ``CorutvError`` / ``ConvergenceError`` (errors.py:4-18),
    so a caller's ``except corutv.errors.ConvergenceError`` (or the
    reference tests' ``pytest.raises``) catches what the device path raises,
    with the same ``residual`` / ``history`` fields.  The raise sites get
    subclasses of both classes (still subclasses of this package's own, so
    ``except paper_1906_04572_b200.CorutvError`` keeps working).
    Idempotent; False if the reference module lacks the classes."""
    import sys

    from . import _lib, errors as ours, rpca as _rpca

    ref_base = getattr(errs, "CorutvError", None)
    ref_conv = getattr(errs, "ConvergenceError", None)
    if ref_base is None or ref_conv is None:
        return False
    if issubclass(_lib.ConvergenceError, ref_conv) and issubclass(_lib.CorutvError, ref_base):
        return True
    base = type("CorutvError", (ours.CorutvError, ref_base), {"__module__": ours.__name__})
    conv = type("ConvergenceError", (ours.ConvergenceError, ref_conv), {"__module__": ours.__name__})
    for mod in (_lib, _rpca, sys.modules[__name__]):
        if hasattr(mod, "CorutvError"):
            mod.CorutvError = base
        if hasattr(mod, "ConvergenceError"):
            mod.ConvergenceError = conv
    return True


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
    try:
        errs = importlib.import_module(f"{ref_pkg.__name__}.errors")
    except ImportError:
        errs = None
    if errs is not None and _adopt_reference_errors(errs):
        done.append(f"{errs.__name__}.CorutvError/ConvergenceError (base classes)")
    for name, obj in (("corutv", corutv), ("alm_corutv", alm_corutv)):
        setattr(ref_pkg, name, obj)
        done.append(f"{ref_pkg.__name__}.{name}")
    for name, obj in (("sor_svd", sor_svd), ("tsr_svd", tsr_svd), ("inexact_alm", inexact_alm), ("svt", svt)):
        if hasattr(ref_pkg, name):
            setattr(ref_pkg, name, obj)
            done.append(f"{ref_pkg.__name__}.{name}")
    return done
