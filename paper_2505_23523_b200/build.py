"""Build libstragglar.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libstragglar.so")
SOURCES = ["api.cu", "kernels.cu", "kernels_i32.cu", "kernels_f32.cu", "kernels_bf16.cu", "nvls.cu", "schedule.cpp"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
    "-Xptxas", "-v",
    "-shared", "-cudart", "static",
]


def source_digest(defines=()) -> str:
    """Content hash of everything the library is built from (mtimes do not
    survive the copy to the GPU box, contents do)."""
    import hashlib

    h = hashlib.sha256()
    deps = sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC))
    deps += [os.path.join(HERE, "..", "include", "stragglar.h"), os.path.abspath(__file__)]
    for d in deps:
        if os.path.isfile(d):
            h.update(os.path.basename(d).encode())
            h.update(open(d, "rb").read())
    h.update(repr((FLAGS, tuple(defines))).encode())
    return h.hexdigest()


def device_digest() -> str:
    """Content hash of the device code (kernels, device primitives, launch plan
    layout): an ncu DRAM-traffic figure is only valid for the kernels it was
    captured on (profiles/latest_traffic.json, bench.py)."""
    import hashlib

    h = hashlib.sha256()
    for f in sorted(os.listdir(CSRC)):
        if f.startswith("kernels") or f in ("device.cuh", "plan.h", "schedule.h"):
            h.update(f.encode())
            h.update(open(os.path.join(CSRC, f), "rb").read())
    return h.hexdigest()[:16]


def needs_build() -> bool:
    stamp = LIB + ".sha256"
    if not os.path.exists(LIB) or not os.path.exists(stamp):
        return True
    return open(stamp).read().strip() != source_digest()


def build(force: bool = False, verbose: bool = False, defines=(), out: str = LIB) -> str:
    """defines: extra -D tuning knobs (STRAGGLAR_STAGES, STRAGGLAR_STAGE_BYTES,
    STRAGGLAR_THREADS, STRAGGLAR_MIN_BLOCKS) for tuning variants built to `out`."""
    if not force and not defines and out == LIB and not needs_build():
        return LIB
    tmp = f"{out}.{os.getpid()}.tmp"        # concurrent builders (torchrun ranks) never share a temp file
    import tempfile
    from concurrent.futures import ThreadPoolExecutor

    objdir = tempfile.mkdtemp(prefix="stragglar_build_")
    compile_flags = [f for f in FLAGS if f not in ("-shared",)]
    defs = [f"-D{d}" for d in defines]

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        r = subprocess.run([NVCC, *compile_flags, *defs, "-c", os.path.join(CSRC, src), "-o", obj],
                           capture_output=True, text=True)
        return src, obj, r

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        results = list(ex.map(compile_one, SOURCES))
    errs = [r for _, _, r in results if r.returncode != 0]
    if errs:
        for r in errs:
            sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libstragglar.so")
    link = subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static",
                           *[o for _, o, _ in results], "-o", tmp], capture_output=True, text=True)
    if link.returncode != 0:
        sys.stderr.write(link.stdout + link.stderr)
        raise RuntimeError("nvcc failed linking libstragglar.so")

    class _Res:
        stderr = "".join(r.stderr for _, _, r in results)

    res = _Res()
    if out == LIB:
        with open(os.path.join(HERE, "ptxas_report.txt"), "w") as f:
            f.write(res.stderr)
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(tmp, out)
    if out == LIB:
        with open(LIB + ".sha256", "w") as f:
            f.write(source_digest())
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
