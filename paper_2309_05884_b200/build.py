"""In-tree build of the CUDA library (nvcc, sm_100a only)."""

from __future__ import annotations

import os
import re
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SOURCES = [os.path.join(HERE, "csrc", f) for f in ("engine.cu", "large.cu", "basis.cu", "trotter.cu")]
DEPS = [os.path.join(HERE, "csrc", f) for f in os.listdir(os.path.join(HERE, "csrc"))] + [
    os.path.join(HERE, "..", "include", "symqoc_b200.h")
]
OUT = os.path.join(HERE, "libsymqoc_b200.so")
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC",
]


def up_to_date() -> bool:
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(p) <= t for p in DEPS)


def _includes(path: str, seen: set) -> set:
    """Local (quoted) include closure of a source file."""
    if path in seen or not os.path.exists(path):
        return seen
    seen.add(path)
    for line in open(path):
        m = re.match(r'\s*#include\s+"([^"]+)"', line)
        if m:
            for base in (os.path.dirname(path), os.path.join(HERE, "..", "include")):
                cand = os.path.normpath(os.path.join(base, m.group(1)))
                if os.path.exists(cand):
                    _includes(cand, seen)
                    break
    return seen


def _obj_stale(src: str, obj: str) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(p) > t for p in _includes(src, set()))


def build(force: bool = False, verbose: bool = False) -> str:
    if force or not up_to_date():
        nvcc = os.environ.get("NVCC", "nvcc")
        objs, procs = [], []
        for src in SOURCES:  # compile translation units in parallel
            obj = os.path.join(HERE, "csrc", os.path.basename(src) + ".o")
            objs.append(obj)
            if not force and not _obj_stale(src, obj):
                continue
            cmd = [nvcc, *NVCC_FLAGS, *os.environ.get("SQOC_NVCC_EXTRA", "").split(), "-c", "-o", obj, src]
            if verbose:
                print(" ".join(cmd), flush=True)
            procs.append(subprocess.Popen(cmd))
        for pr in procs:
            if pr.wait() != 0:
                raise RuntimeError("nvcc failed")
        link = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", OUT + ".tmp", *objs, "-lcudart"]
        if verbose:
            print(" ".join(link), flush=True)
        subprocess.run(link, check=True)
        os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    print(build(force=True, verbose=True))
