"""The engine's trig (csrc/pf_trig.h) through its CPU twin: correctly
rounded (checked against mpmath) and therefore equal to glibc wherever glibc
is correctly rounded.  The GPU build is checked bit-identical to this twin in
test_gpu_trig (tests/test_gpu_parity.py)."""

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np
import pytest

HERE = Path(__file__).resolve().parent


def build_twin(tmpdir: Path) -> C.CDLL:
    so = tmpdir / "trig_twin.so"
    subprocess.run(["/usr/bin/gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
                    "-shared", "-std=c11", str(HERE / "native" / "trig_twin.c"), "-o", str(so),
                    "-lm"], check=True)
    lib = C.CDLL(str(so))
    lib.twin_sincos.argtypes = [C.c_void_p] * 3 + [C.c_int64]
    return lib


def twin_sincos(lib, x):
    x = np.ascontiguousarray(x, dtype=np.float64)
    s, c = np.zeros_like(x), np.zeros_like(x)
    lib.twin_sincos(x.ctypes.data, s.ctypes.data, c.ctypes.data, x.size)
    return s, c


def sample(n=20000, seed=1):
    rng = np.random.default_rng(seed)
    return np.concatenate([rng.normal(0, 0.3, n), rng.uniform(-3.3, 3.3, n // 2),
                           rng.uniform(-200, 200, n // 4), rng.uniform(-1e-4, 1e-4, 500),
                           [0.0, -0.0, np.pi / 4, -np.pi / 2, np.pi, 1e6, 5e-324]])


@pytest.fixture(scope="module")
def twin(tmp_path_factory):
    return build_twin(tmp_path_factory.mktemp("twin"))


def test_twin_correctly_rounded(twin):
    mpmath = pytest.importorskip("mpmath")
    mpmath.mp.prec = 120
    x = sample(8000)
    s, c = twin_sincos(twin, x)
    cs = np.array([float(mpmath.sin(mpmath.mpf(float(v)))) for v in x])
    cc = np.array([float(mpmath.cos(mpmath.mpf(float(v)))) for v in x])
    # near-correct rounding: a handful of near-midpoint misses at most
    assert np.sum(s != cs) <= 2 and np.sum(c != cc) <= 2
    ulp = np.abs(s.view(np.int64) - cs.view(np.int64)).max()
    assert ulp <= 1
    assert np.signbit(s[np.flatnonzero((x == 0) & np.signbit(x))]).all()


def test_twin_agrees_with_glibc(twin):
    import oracle

    x = sample(40000, seed=2)
    s, c = twin_sincos(twin, x)
    gs, gc = oracle.libm_sincos(x)
    assert np.mean(s == gs) > 0.995 and np.mean(c == gc) > 0.998


def test_special_values(twin):
    x = np.array([np.inf, -np.inf, np.nan, 2.0 ** 30])
    s, c = twin_sincos(twin, x)
    assert np.isnan(s[:3]).all() and np.isnan(c[:3]).all()
    assert s[3] == np.sin(2.0 ** 30) or abs(s[3] - np.sin(2.0 ** 30)) < 1e-15


def test_twin_odd_even_bit_for_bit(twin):
    """sin(-x) == -sin(x) and cos(-x) == cos(x) exactly, fast and slow paths:
    the kernels evaluate a branch's k terminal at -thk (pf_eval.cu inc_terms)."""
    x = np.concatenate([sample(200000, seed=5), [2.0 ** 20, 3.5e6, 2.0 ** 40, 1e300]])
    s, c = twin_sincos(twin, x)
    sn, cn = twin_sincos(twin, -x)
    assert np.array_equal((-s).view(np.int64), sn.view(np.int64))
    assert np.array_equal(c.view(np.int64), cn.view(np.int64))
