"""Build libcakf.so in-tree with nvcc for sm_100a (no JIT, no torch extension machinery).

    python -m paper_2405_08971_b200.build          # or __graft_entry__.build()
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libcakf.so")
SOURCES = ["kernels_gram.cu", "kernels_gram_tc.cu", "kernels_gemm_tc.cu", "kernels_gemm_i8.cu", "kd_order.cu", "kernels_step.cu", "kernels_eig.cu",
           "kernels_gemm_f64.cu", "kernels_peak.cu", "cakf_api.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
try:  # NCCL as bundled with torch (nvidia-nccl wheel): headers + libnccl.so.2
    import nvidia.nccl as _nccl
    NCCL_DIR = os.path.dirname(_nccl.__file__) if _nccl.__file__ else list(_nccl.__path__)[0]
except Exception:  # pragma: no cover
    NCCL_DIR = "/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl"


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "cakf.h")]
    return any(os.path.getmtime(p) > t for p in deps if os.path.exists(p))


def build(force: bool = False, verbose: bool = False, extra: list[str] | None = None, out: str | None = None) -> str:
    """extra / out: experiment builds (extra nvcc -D flags, a separate library path for CAKF_LIB A/B runs)."""
    lib = out or LIB
    if not force and not extra and not _stale():
        return LIB
    objs = []
    build_dir = os.path.join(HERE, "build" if not out else "build_" + os.path.basename(out).replace(".so", ""))
    os.makedirs(build_dir, exist_ok=True)
    common = [nvcc(), "-O3", "-std=c++17", *ARCH, "-lineinfo", "-Xcompiler", "-fPIC",
              "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", os.path.join(NCCL_DIR, "include"),
              "-Xptxas", "-v" if verbose else "-O3", *(extra or [])]
    procs = []
    for src in SOURCES:
        obj = os.path.join(build_dir, src.replace(".cu", ".o"))
        objs.append(obj)
        cmd = common + ["-c", os.path.join(CSRC, src), "-o", obj]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
    for cmd, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + out)
        if verbose and out:
            print(out)
    tmp = lib + ".tmp"
    nccl_lib = os.path.join(NCCL_DIR, "lib")
    link = [nvcc(), "-shared", *ARCH, "-o", tmp, *objs, "-lcusolver", "-L", nccl_lib, "-l:libnccl.so.2",
            "-Xlinker", "-rpath,/usr/local/cuda/lib64", "-Xlinker", "-rpath," + nccl_lib]
    r = subprocess.run(link, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
    if r.returncode != 0:
        raise RuntimeError("link failed:\n" + " ".join(link) + "\n" + r.stdout)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    _extra = [a for a in sys.argv[1:] if a.startswith("-D")]
    _out = next((a[len("--out="):] for a in sys.argv[1:] if a.startswith("--out=")), None)
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, extra=_extra, out=_out))
