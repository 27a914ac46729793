"""Builds libtoposmooth_b200.so in-tree with nvcc for sm_100a (translation
units compiled in parallel, then linked).

    python -m paper_1603_09337_b200.build [--verbose]
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "build_obj")
LIB = os.path.join(HERE, "libtoposmooth_b200.so")
SOURCES = ["ts_hasf_8h.cu", "ts_hasf_4h.cu", "ts_hasf_8g.cu", "ts_hasf_4g.cu", "ts_hasf_8h256.cu",
           "ts_hasf_4h256.cu", "ts_hasf_8g1024.cu", "ts_hasf_4g1024.cu", "ts_hasf.cu", "ts_edt.cu", "ts_ccl.cu", "ts_p4.cu", "ts_api.cu", "ts_hostpack.cpp"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         *os.environ.get("TS_NVCC_EXTRA", "").split()]   # TS_NVCC_EXTRA: extra nvcc flags (A/B builds)


def _deps():
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(HERE, "..", "include", "toposmooth_b200.h"))
    deps.append(os.path.abspath(__file__))
    return [d for d in deps if os.path.exists(d)]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in _deps())


def build(verbose: bool = False, force: bool = False, defines=(), out: str | None = None) -> str:
    """Compile all translation units in parallel and link the shared library.
    `defines` (e.g. ["TS_MIN_BLOCKS=1"]) and `out` build experiment variants.
    Serialised across processes by an flock (torchrun ranks importing a stale
    tree build once; the others wait and then find it current)."""
    import fcntl
    os.makedirs(OBJ, exist_ok=True)
    with open(os.path.join(OBJ, ".build.lock"), "w") as lock:
        fcntl.flock(lock, fcntl.LOCK_EX)
        try:
            return _build_locked(verbose, force, defines, out)
        finally:
            fcntl.flock(lock, fcntl.LOCK_UN)


def _build_locked(verbose, force, defines, out):
    lib = out or LIB
    if not force and not defines and out is None and not needs_build():
        return LIB
    obj_dir = OBJ if not defines else OBJ + "_" + "_".join(d.replace("=", "") for d in defines)
    os.makedirs(obj_dir, exist_ok=True)
    procs = []
    for src in SOURCES:
        obj = os.path.join(obj_dir, os.path.splitext(src)[0] + ".o")
        extra = ["-Xcompiler", "-fopenmp"] if src.endswith(".cpp") else []   # host packing threads
        cmd = [NVCC, *ARCH, *FLAGS, *extra, *[f"-D{d}" for d in defines], "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            cmd += ["-Xptxas", "-v"]
        procs.append((src, obj, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT,
                                                 text=True)))
    objs, failed = [], []
    for src, obj, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            failed.append(src)
            sys.stderr.write(out)
        elif verbose:
            sys.stderr.write(out)
        objs.append(obj)
    if failed:
        raise RuntimeError(f"nvcc failed on {failed}")
    tmp = f"{lib}.tmp{os.getpid()}"   # per-process: ranks never share a temp file
    res = subprocess.run([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lgomp"], capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc link failed for libtoposmooth_b200.so")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--define", action="append", default=[])
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    print(build(verbose=a.verbose, force=True, defines=a.define, out=a.out))
