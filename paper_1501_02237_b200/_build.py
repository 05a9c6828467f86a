"""Build libbdeg.so in-tree with nvcc for sm_100a (no JIT cache, no CPU path)."""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libbdeg.so")
# the four bdeg_enum_t*.cu hold the k_enumerate instantiations of one arithmetic
# tier each: compiled in parallel (objects), then linked
SOURCES = ["bdeg_enum_t0.cu", "bdeg_enum_t1.cu", "bdeg_enum_t2.cu", "bdeg_enum_t3.cu", "bdeg_kernels.cu",
           "bdeg_walk.cu", "bdeg_rank.cu", "bdeg_capi.cpp", "frontend.cpp"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "bdeg.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build_lib(force: bool = False, verbose: bool = False, out: str = LIB, defines=()) -> str:
    if out == LIB and not force and not _stale():
        return LIB
    import tempfile
    from concurrent.futures import ThreadPoolExecutor
    flags = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
             "-Xptxas", "-v" if verbose else "-O3", "-I", os.path.join(ROOT, "include"),
             *[f"-D{d}" for d in defines]]
    with tempfile.TemporaryDirectory(prefix="bdeg_build_") as tmp:
        objs = [os.path.join(tmp, f + ".o") for f in SOURCES]

        def compile_one(i):
            subprocess.check_call([NVCC, *flags, "-c", "-o", objs[i], os.path.join(CSRC, SOURCES[i])])

        # the largest translation units first
        order = sorted(range(len(SOURCES)), key=lambda i: -os.path.getsize(os.path.join(CSRC, SOURCES[i])))
        with ThreadPoolExecutor(max_workers=max(1, min(len(SOURCES), os.cpu_count() or 1))) as ex:
            list(ex.map(compile_one, order))
        subprocess.check_call([NVCC, *ARCH, "-shared", "-o", out + ".tmp", *objs, "-lcudart"])
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    import sys
    print(build_lib(force=True, verbose="-v" in sys.argv))
