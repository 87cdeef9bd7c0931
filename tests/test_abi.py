"""The C-ABI library builds for sm_100a, loads, and exports include/pfgpu.h.

No compute calls here (no GPU in the build container)."""

import re
import subprocess
from pathlib import Path

import pytest

from paper_2011_11880_b200 import _abi

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "pfgpu.h"


def header_symbols():
    text = HEADER.read_text()
    return set(re.findall(r"PF_API\s+[\w\s\*]+?\b(pf_\w+)\s*\(", text))


@pytest.fixture(scope="module")
def built():
    from paper_2011_11880_b200.build import build

    return build()


def test_header_and_binding_agree():
    assert header_symbols() == set(_abi.EXPORTED)


def test_library_exports_every_symbol(built):
    out = subprocess.run(["nm", "-D", "--defined-only", str(built)], capture_output=True,
                         text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    assert header_symbols() <= exported
    # nothing else leaks (hidden visibility)
    assert {s for s in exported if s.startswith("pf_")} == header_symbols()


def test_library_loads_without_gpu(built):
    lib = _abi.lib()
    assert lib.pf_version() == 1
    assert lib.pf_launch_count() >= 0


def test_library_is_sm100a(built):
    out = subprocess.run(["cuobjdump", "--list-elf", str(built)], capture_output=True,
                         text=True, check=True).stdout
    assert "sm_100a" in out


def test_plan_create_rejects_bad_topology_before_touching_gpu(built):
    """Argument validation happens on the host (pf_plan_create -> PF_EINVAL)."""
    import ctypes as C

    import numpy as np

    from paper_2011_11880_b200.system_model import build_system
    from paper_2011_11880_b200 import synth

    s = build_system(synth.synth_case(5, 6, seed=1, pq_frac=0.5, pv_frac=0.2))
    t, keep = _abi.topology(s)
    bad_h = np.array(s.lines.bus_h, dtype=np.int32)
    bad_h[0] = s.lines.bus_k[0]  # self-loop
    t.bus_h = bad_h.ctypes.data_as(C.POINTER(C.c_int32))
    h = C.c_void_p()
    rc = _abi.lib().pf_plan_create(C.byref(t), C.byref(h))
    assert rc == _abi.PF_EINVAL
    assert b"self-loop" in _abi.lib().pf_last_error()
    bad_h[0] = 99
    rc = _abi.lib().pf_plan_create(C.byref(t), C.byref(h))
    assert rc == _abi.PF_EINVAL
    assert b"bus index" in _abi.lib().pf_last_error()
    del keep


def test_host_side_argument_checks_without_gpu(built):
    """NULL / negative arguments are rejected on the host with PF_EINVAL and a
    message, before any CUDA call (pflow raises ValueError at bind time)."""
    lib = _abi.lib()
    assert lib.pf_batch_unblock(-1, 4, None, None, 1.0, None) == _abi.PF_EINVAL
    assert b"negative" in lib.pf_last_error()
    assert lib.pf_batch_unblock(2, 4, None, None, 1.0, None) == _abi.PF_EINVAL
    assert b"NULL" in lib.pf_last_error()
    assert lib.pf_batch_update(2, 4, None, None, None, None) == _abi.PF_EINVAL
    assert lib.pf_eval(None, None, None, None, None, None) == _abi.PF_EINVAL
    assert lib.pf_plan_destroy(None) in (_abi.PF_OK, _abi.PF_EINVAL)
    with pytest.raises(ValueError):
        _abi.check(_abi.PF_EINVAL)
    with pytest.raises(RuntimeError):
        _abi.check(_abi.PF_ECUDA)
