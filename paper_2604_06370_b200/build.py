"""Build libforkkv.so in-tree (sm_100a) with nvcc.

    python -m paper_2604_06370_b200.build [--force]

Every .cu/.cpp under csrc/ is compiled with
    -gencode arch=compute_100a,code=sm_100a -lineinfo -O3
and linked into paper_2604_06370_b200/libforkkv.so (static cudart, so the
library loads on a CPU-only host for the control-plane tests).
"""
from __future__ import annotations

import glob
import hashlib
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libforkkv.so")
OBJ = os.path.join(HERE, "build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", f"-I{ROOT}/include", f"-I{CSRC}"]


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def _headers():
    return sorted(glob.glob(os.path.join(CSRC, "*.hpp")) + glob.glob(os.path.join(ROOT, "include", "*.h")))


def _digest(path: str, extra: bytes = b"") -> str:
    h = hashlib.sha1(extra)
    with open(path, "rb") as f:
        h.update(f.read())
    for hd in _headers():
        with open(hd, "rb") as f:
            h.update(f.read())
    h.update(" ".join(ARCH + COMMON).encode())
    return h.hexdigest()[:16]


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    objs = []
    procs = []
    for src in _sources():
        name = os.path.splitext(os.path.basename(src))[0] + os.path.splitext(src)[1].replace(".", "_")
        obj = os.path.join(OBJ, f"{name}.{_digest(src)}.o")
        objs.append(obj)
        if os.path.exists(obj) and not force:
            continue
        flags = ARCH + COMMON
        if src.endswith(".cu"):
            flags = flags + ["-Xptxas", "-v"] if verbose else flags
        cmd = [NVCC, *flags, "-c", src, "-o", obj]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    for cmd, pr in procs:
        out, _ = pr.communicate()
        if verbose and out:
            sys.stdout.write(out.decode())
        if pr.returncode != 0:
            sys.stderr.write(out.decode())
            raise RuntimeError("nvcc failed: " + " ".join(cmd))
    tmp = OUT + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-Xcompiler", "-fPIC", "-cudart", "static", "-o", tmp, *objs]
    subprocess.check_call(cmd)
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(OUT)
