"""The C-ABI boundary used from plain C (tests/c/abi_client.c, gcc, no
Python in the process): it builds and links against libcorutv_b200.so on
the CPU, and on the GPU its decomposition is bitwise the Python entry's
(same library call) and matches the oracle (sketch.py:182-208)."""

import json
import shutil
import subprocess
from pathlib import Path

import numpy as np
import pytest

import oracle as O

ROOT = Path(__file__).resolve().parents[1]
LIBDIR = ROOT / "paper_1906_04572_b200"
CUDA = Path("/usr/local/cuda")


def _build(tmp_path):
    if not (LIBDIR / "libcorutv_b200.so").exists():
        pytest.skip("library not built")
    if shutil.which("gcc") is None or not (CUDA / "include" / "cuda_runtime.h").exists():
        pytest.skip("gcc / CUDA headers not available")
    exe = tmp_path / "abi_client"
    subprocess.run(["gcc", "-std=c99", "-O2", "-Wall", "-Werror", "-I", str(ROOT / "include"),
                    "-I", str(CUDA / "include"), str(ROOT / "tests" / "c" / "abi_client.c"), "-o", str(exe),
                    "-L", str(LIBDIR), "-lcorutv_b200", "-L", str(CUDA / "lib64"), "-lcudart",
                    f"-Wl,-rpath,{LIBDIR}:{CUDA / 'lib64'}"], check=True)
    return exe


def test_c_client_builds_and_links(tmp_path):
    exe = _build(tmp_path)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout
    assert json.loads(out)["version"] >= 1


@pytest.mark.gpu
@pytest.mark.parametrize("m,n,k,ell,q,variant", [(600, 250, 12, 30, 1, 0), (333, 333, 40, 41, 0, 1)])
def test_c_client_decomposition(tmp_path, m, n, k, ell, q, variant):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1906_04572_b200 as P

    exe = _build(tmp_path)
    g = np.random.Generator(np.random.PCG64(m + n))
    a = g.standard_normal((m, k)) @ g.standard_normal((k, n)) + 1e-6 * g.standard_normal((m, n))
    om = g.standard_normal((n, ell))
    fin, fout = tmp_path / "in.bin", tmp_path / "out.bin"
    with open(fin, "wb") as fh:
        np.array([m, n, ell, q, variant], dtype=np.int64).tofile(fh)
        a.tofile(fh)
        om.tofile(fh)
    res = subprocess.run([str(exe), str(fin), str(fout)], check=True, capture_output=True, text=True, timeout=300)
    line = json.loads(res.stdout.strip().splitlines()[-1])
    assert line["rc"] == 0, line
    raw = np.fromfile(fout, dtype=np.float64)
    passes = int(raw[:1].view(np.int64)[0])
    off = 1
    u = raw[off:off + m * ell].reshape(m, ell); off += m * ell
    t = raw[off:off + ell * ell].reshape(ell, ell); off += ell * ell
    v = raw[off:off + n * ell].reshape(n, ell); off += n * ell
    perm = raw[off:off + ell].view(np.int64)
    # the same library call from Python: bitwise identical
    var = P.VARIANT_EXACT if variant == 0 else P.VARIANT_APPROX
    f = P.corutv(a, P.SketchConfig(ell=ell, q_power=q, variant=var), omega=om)
    assert np.array_equal(u, f.u) and np.array_equal(t, f.t) and np.array_equal(v, f.v)
    assert np.array_equal(perm, np.asarray(f.perm))
    # and the oracle (reference algorithm) to rounding
    ref = O.corutv(a, ell, q, variant=O.VARIANT_EXACT if variant == 0 else O.VARIANT_APPROX, omega=om)
    assert passes == ref["passes"]
    d, dref = np.abs(np.diag(t)), np.abs(np.diag(ref["t"]))
    assert np.abs(d[:k] - dref[:k]).max() <= 1e-9 * dref[0]
    e_ref = np.linalg.norm(a - ref["u"] @ ref["t"] @ ref["v"].T)
    assert abs(line["err"] - e_ref) <= 1e-8 * np.linalg.norm(a)
