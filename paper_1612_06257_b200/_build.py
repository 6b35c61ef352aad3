"""Build the in-tree CUDA library libb200hash.so for sm_100a (nvcc, no GPU needed).

Each translation unit compiles to its own object in parallel (the Sip-family
kernels are one object per variant of csrc/lh_sip_variants.h, from
csrc/lh_sip_variant.cu), then nvcc links the shared library.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "build")
SO = os.path.join(HERE, "libb200hash.so")
SOURCES = ["lh_engine.cu", "lh_synth.cu", "lh_stream.cu", "lh_quality.cu", "lh_state.cu",
           "lh_plan.cu"]
# (tag, C, D, TREE) -- must match LH_SIP_VARIANTS in csrc/lh_sip_variants.h
SIP_VARIANTS = [("s24", 2, 4, 0), ("s13", 1, 3, 0), ("s00", 0, 0, 0),
                ("t24", 2, 4, 1), ("t13", 1, 3, 1), ("t00", 0, 0, 1)]
HEADERS = ["lh_device.cuh", "lh_tma.cuh", "lh_reader.cuh", "lh_host.cuh", "lh_mix.cuh",
           "lh_stream.cuh", "lh_kernels.cuh", "lh_sip_variants.h", "lh_sip_variant.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = [
    "-O3",
    "-std=c++17",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo",
    "-Xcompiler", "-fPIC,-O2",
    "--expt-relaxed-constexpr",
]


def _units():
    """(object path, source path, extra flags) per translation unit."""
    units = [(os.path.join(OBJ, s[:-3] + ".o"), os.path.join(CSRC, s), []) for s in SOURCES]
    for tag, c, d, tree in SIP_VARIANTS:
        units.append((os.path.join(OBJ, f"lh_sip_{tag}.o"), os.path.join(CSRC, "lh_sip_variant.cu"),
                      [f"-DLH_VAR_TAG={tag}", f"-DLH_VAR_C={c}", f"-DLH_VAR_D={d}",
                       f"-DLH_VAR_TREE={tree}"]))
    return units


def _inputs():
    root = os.path.dirname(HERE)
    files = [os.path.join(CSRC, s) for s in SOURCES + HEADERS]
    files.append(os.path.join(root, "include", "lanehash_b200.h"))
    files.append(os.path.abspath(__file__))
    return files


def stale() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    return any(os.path.getmtime(f) > t for f in _inputs())


def build(force: bool = False, verbose: bool = False, so: str = SO, obj: str = OBJ) -> str:
    """Compile and link.  ``so``/``obj`` redirect an A/B variant build
    (LH_NVCC_EXTRA=-D...) away from the in-tree library."""
    if not force and so == SO and not stale():
        return SO
    os.makedirs(obj, exist_ok=True)
    extra = os.environ.get("LH_NVCC_EXTRA", "").split()
    if verbose:
        extra += ["-Xptxas", "-v"]

    def compile_one(unit):
        obj, src, defs = unit
        cmd = [NVCC, *FLAGS, *extra, *defs, "-c", src, "-o", obj]
        return subprocess.run(cmd, cwd=CSRC, capture_output=True, text=True), cmd

    units = [(os.path.join(obj, os.path.basename(o)), src, defs) for o, src, defs in _units()]
    with ThreadPoolExecutor(max_workers=min(len(units), os.cpu_count() or 4)) as pool:
        results = list(pool.map(compile_one, units))
    for r, cmd in results:
        if verbose or r.returncode:
            sys.stderr.write(r.stdout + r.stderr)
        if r.returncode:
            raise subprocess.CalledProcessError(r.returncode, cmd, r.stdout, r.stderr)
    link = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-Xcompiler", "-fPIC",
            "-o", so + ".tmp", *[u[0] for u in units]]
    subprocess.run(link, check=True, cwd=CSRC)
    os.replace(so + ".tmp", so)
    return so


if __name__ == "__main__":
    import argparse

    ap = argparse.ArgumentParser()
    ap.add_argument("-v", action="store_true")
    ap.add_argument("--so", default=SO)
    ap.add_argument("--obj", default=OBJ)
    a = ap.parse_args()
    print(build(force=True, verbose=a.v, so=os.path.abspath(a.so), obj=os.path.abspath(a.obj)))
