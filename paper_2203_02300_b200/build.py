"""Builds libdco_gpu.so in-tree: every csrc/*.cu compiled for sm_100a only.

nvcc flags:
  -gencode arch=compute_100a,code=sm_100a   B200 only (no PTX fallback, no other arch)
  --fmad=false                              no FMA contraction: float/double results
                                            round exactly like the reference's x86-64
                                            build; fused ops are
                                            written explicitly (__fma_rn) where the
                                            replicated glibc code fuses
  -lineinfo                                 ncu source attribution
Objects are compiled in parallel and cached by content hash under build/.
"""
import hashlib
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(HERE, "libdco_gpu.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ARCH + [
    "-O3",
    "-std=c++17",
    "--fmad=false",
    "-lineinfo",
    "-Xcompiler",
    "-fPIC,-fvisibility=hidden,-ffp-contract=off",
    "-Xptxas",
    "-warn-spills",
    "-I" + CSRC,
    "-I" + os.path.join(ROOT, "include"),
    "--expt-relaxed-constexpr",
]


def _sources():
    return sorted(f for f in os.listdir(CSRC) if f.endswith(".cu"))


def _digest(src):
    h = hashlib.sha256()
    h.update(" ".join(FLAGS).encode())
    for name in sorted(os.listdir(CSRC)):
        if name.endswith((".cuh", ".h", ".inc")):
            h.update(open(os.path.join(CSRC, name), "rb").read())
    h.update(open(os.path.join(ROOT, "include", "dco_gpu.h"), "rb").read())
    h.update(open(os.path.join(CSRC, src), "rb").read())
    return h.hexdigest()[:16]


def _compile(src):
    obj = os.path.join(OBJ, "%s.%s.o" % (src[:-3], _digest(src)))
    if not os.path.exists(obj):
        cmd = [NVCC] + FLAGS + ["-c", os.path.join(CSRC, src), "-o", obj + ".tmp"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed for %s:\n%s\n%s" % (src, r.stdout, r.stderr))
        if r.stderr.strip():
            sys.stderr.write(r.stderr)
        os.replace(obj + ".tmp", obj)
        # drop this source's stale objects (older digests)
        stem = src[:-3] + "."
        for f in os.listdir(OBJ):
            if f.startswith(stem) and f.endswith(".o") and os.path.join(OBJ, f) != obj:
                os.remove(os.path.join(OBJ, f))
    return obj


def build(verbose=True):
    os.makedirs(OBJ, exist_ok=True)
    srcs = _sources()
    with ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(_compile, srcs))
    cmd = [NVCC] + ARCH + ["-shared", "-o", LIB + ".tmp"] + objs + ["-lcudart_static", "-lrt", "-ldl", "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("link failed:\n%s\n%s" % (r.stdout, r.stderr))
    os.replace(LIB + ".tmp", LIB)
    if verbose:
        print("built", LIB)
    return LIB


if __name__ == "__main__":
    build()
