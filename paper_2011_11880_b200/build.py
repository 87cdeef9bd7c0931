"""Build libpfgpu.so (sm_100a) in-tree with nvcc.

pf_eval.cu is compiled with -fmad=false so its fp64 arithmetic rounds where
the reference's wf1 rounds (see the file header); pf_plan.cu (symbolic build,
C ABI) uses default flags.  Static cudart; the library exports only the
extern "C" symbols of include/pfgpu.h.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OUT = PKG / "libpfgpu.so"
BUILD = ROOT / "build"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-fvisibility=hidden",
          "-I", str(ROOT / "include"), *ARCH]
UNITS = {
    "pf_eval.cu": ["-fmad=false"],
    "pf_plan.cu": [],
    "pf_lu.cu": [],
}


def source_hash() -> str:
    """Hash of every kernel source and the compile flags: identifies the build
    an ncu capture was taken from (profiles/traffic.json)."""
    import hashlib

    h = hashlib.sha256()
    for p in sorted([*CSRC.glob("*.cu"), *CSRC.glob("*.h"), *CSRC.glob("*.cuh"),
                     ROOT / "include" / "pfgpu.h"]):
        h.update(p.name.encode())
        h.update(p.read_bytes())
    # flags without the checkout's absolute path (the GPU box runs a copy elsewhere)
    h.update(repr(([f.replace(str(ROOT), "<root>") for f in COMMON], UNITS)).encode())
    return h.hexdigest()[:16]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (Path(cand).exists() or cand == "nvcc"):
            return cand
    raise RuntimeError("nvcc not found")


def build_variant(name: str, defines: list[str]) -> Path:
    """Dev tool: build/var/<name>.so with extra -D flags (A/B kernel timing)."""
    out_dir = BUILD / "var"
    out_dir.mkdir(parents=True, exist_ok=True)
    objs = []
    for src, extra in UNITS.items():
        o = out_dir / f"{name}.{src}.o"
        subprocess.run([nvcc(), *COMMON, *extra, *[f"-D{d}" for d in defines], "-c",
                        str(CSRC / src), "-o", str(o)], check=True)
        objs.append(o)
    lib = out_dir / f"{name}.so"
    subprocess.run([nvcc(), *ARCH, "-shared", "-o", str(lib), *map(str, objs), "-cudart",
                    "static"], check=True)
    return lib


def build(verbose: bool = False, force: bool = False) -> Path:
    BUILD.mkdir(exist_ok=True)
    objs = []
    deps = [*CSRC.glob("*.h"), *CSRC.glob("*.cuh"), ROOT / "include" / "pfgpu.h"]
    for src, extra in UNITS.items():
        s = CSRC / src
        o = BUILD / (src + ".o")
        objs.append(o)
        newest = max(p.stat().st_mtime for p in [s, *deps])
        if not force and o.exists() and o.stat().st_mtime >= newest:
            continue
        cmd = [nvcc(), *COMMON, *extra, "-Xptxas", "-v" if verbose else "-O3", "-c", str(s),
               "-o", str(o)]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
    if force or not OUT.exists() or OUT.stat().st_mtime < max(o.stat().st_mtime for o in objs):
        cmd = [nvcc(), *ARCH, "-shared", "-o", str(OUT), *map(str, objs), "-cudart", "static"]
        subprocess.run(cmd, check=True)
    return OUT


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--variant":   # --variant NAME [DEFINE ...]
        print(build_variant(sys.argv[2], sys.argv[3:]))
    else:
        build(verbose="-v" in sys.argv, force="-f" in sys.argv)
        print(OUT)
