"""C-ABI boundary checks that need no GPU: the in-tree library loads and
exports every symbol include/corutv_b200.h declares, with the ctypes
signatures the host layer uses; the product path fails loudly without a
device (no CPU fallback)."""

import re
import subprocess
from pathlib import Path

import pytest

from paper_1906_04572_b200 import _lib

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "corutv_b200.h"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = re.findall(r"^\s*(?:[A-Za-z_][\w\s\*]*?)\b(corutv_\w+)\s*\(", text, flags=re.M)
    return sorted(set(n for n in names if n != "corutv_allreduce_fn"))


def test_header_declares_the_hot_path():
    names = declared_functions()
    for must in ("corutv_decompose", "corutv_alm_update", "corutv_spectral_norm",
                 "corutv_lowrank", "corutv_lowrank_error", "corutv_gemm", "corutv_set_comm"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = _lib.load_library()
    for name in declared_functions():
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"{name} has no ctypes signature"
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (corutv_\w+)", out))
    assert set(declared_functions()) <= exported


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_version_without_gpu():
    assert _lib.load_library().corutv_version() >= 100


def test_status_mapping():
    from paper_1906_04572_b200.errors import ConvergenceError, CorutvError

    with pytest.raises(ValueError):
        _lib.check(_lib.ERR_SHAPE)
    with pytest.raises(ValueError):
        _lib.check(_lib.ERR_NONFINITE)
    with pytest.raises(ConvergenceError):
        _lib.check(_lib.ERR_CONVERGENCE)
    with pytest.raises(CorutvError):
        _lib.check(_lib.ERR_CUDA)
    _lib.check(_lib.OK)


def test_no_cpu_fallback_without_device():
    import numpy as np
    import torch

    import paper_1906_04572_b200 as P

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(_lib.DeviceUnavailable):
        P.corutv(np.ones((4, 3)), P.SketchConfig(ell=2))
    with pytest.raises(_lib.DeviceUnavailable):
        P.alm_corutv(np.ones((4, 4)), P.AlmConfig(ell=2))


def test_product_never_imports_oracle():
    pkg = ROOT / "paper_1906_04572_b200"
    for f in pkg.rglob("*.py"):
        src = f.read_text()
        assert "import oracle" not in src and "from oracle" not in src, f
