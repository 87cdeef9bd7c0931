"""The engine's trig (csrc/pf_trig.h) through its CPU twin: bit-identical to
the live glibc libm's sin and cos, which is what the reference's wf1 calls
(pflow kernels.py:84-86 -> @llvm.sin/cos.f64 -> libm).  The GPU build is
checked bit-identical to this twin and to libm in test_gpu_trig
(tests/test_gpu_parity.py).  scripts/trig/glibc_campaign.c runs the same
comparison over 2e9 arguments (profiles/r02_trig_campaign.md)."""

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np
import pytest

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent


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
    """Power-flow angle differences, the middle and reduced ranges, tiny
    arguments, the neighbourhoods of every range limit and table node, and
    special values."""
    rng = np.random.default_rng(seed)
    lims = np.array([2.0 ** -27, 2.0 ** -26, 0.126, 0.85546875, float.fromhex("0x1.368fdp+1"),
                     float.fromhex("0x1.921fbp+26"), np.pi / 2, np.pi, 3 * np.pi / 4])
    nodes = np.concatenate([lims, np.arange(1, 110) / 128.0, np.arange(0, 110) / 128.0 + 1 / 256])
    near = (nodes[rng.integers(0, nodes.size, n // 4)].view(np.int64)
            + rng.integers(-64, 65, n // 4)).view(np.float64)
    x = np.concatenate([rng.normal(0, 0.2 * np.sqrt(2), n), rng.normal(0, 1.0, n // 2),
                        rng.uniform(-4, 4, n // 2), rng.uniform(-200, 200, n // 4),
                        rng.uniform(-1e8, 1e8, n // 8), rng.uniform(-1e-4, 1e-4, 500),
                        rng.uniform(-1e-8, 1e-8, 500), near, -near,
                        [0.0, -0.0, np.pi / 4, -np.pi / 2, np.pi, 1e6, 5e-324]])
    return x


@pytest.fixture(scope="module")
def twin(tmp_path_factory):
    return build_twin(tmp_path_factory.mktemp("twin"))


def test_twin_bit_identical_to_glibc(twin):
    import oracle

    x = sample(400000, seed=2)
    s, c = twin_sincos(twin, x)
    gs, gc = oracle.libm_sincos(x)           # libm sin() and cos(), called separately
    assert np.array_equal(s.view(np.int64), gs.view(np.int64))
    assert np.array_equal(c.view(np.int64), gc.view(np.int64))


def test_glibc_campaign_program(tmp_path):
    """The campaign tool itself (8 distributions x 1M arguments, sin and cos
    through volatile pointers, sincos as a cross-check): exit 0 = no
    mismatch."""
    exe = tmp_path / "campaign"
    subprocess.run(["/usr/bin/gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-o", str(exe),
                    str(ROOT / "scripts" / "trig" / "glibc_campaign.c"), "-lm"], check=True)
    r = subprocess.run([str(exe), "1000000", "5"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout
    assert "TOTAL 8000000 arguments (x2 functions), 0 mismatches" in r.stdout


def test_special_values(twin):
    x = np.array([np.inf, -np.inf, np.nan, 2.0 ** 30, 0.0, -0.0, 1e-300, -1e-300])
    s, c = twin_sincos(twin, x)
    assert np.isnan(s[:3]).all() and np.isnan(c[:3]).all()
    assert s[3] == np.sin(2.0 ** 30) or abs(s[3] - np.sin(2.0 ** 30)) < 1e-15
    assert np.array_equal(s[4:].view(np.int64), x[4:].view(np.int64))   # sin x = x, signed
    assert (c[4:] == 1.0).all()


def test_twin_odd_even_bit_for_bit(twin):
    """sin(-x) == -sin(x) and cos(-x) == cos(x) exactly, every range: the
    kernels evaluate a branch's k terminal at -thk (pf_eval.cu inc_terms)."""
    x = np.concatenate([sample(200000, seed=5), [2.0 ** 20, 3.5e6, 2.0 ** 40, 1e300]])
    s, c = twin_sincos(twin, x)
    sn, cn = twin_sincos(twin, -x)
    assert np.array_equal((-s).view(np.int64), sn.view(np.int64))
    assert np.array_equal(c.view(np.int64), cn.view(np.int64))
