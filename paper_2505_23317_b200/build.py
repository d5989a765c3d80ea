"""Build libcfdetr.so in-tree with nvcc for sm_100a (no torch extension machinery).

`python -m paper_2505_23317_b200.build` or `build()` from __graft_entry__.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libcfdetr.so")
LIB_DBG = os.path.join(HERE, "libcfdetr_dbg.so")
SOURCES = ["cfdetr.cu"]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O2",
    "--expt-relaxed-constexpr",
    "-Xptxas", "-v",
]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _newest_src_mtime() -> float:
    paths = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [
        os.path.join(ROOT, "include", f) for f in os.listdir(os.path.join(ROOT, "include"))]
    return max(os.path.getmtime(p) for p in paths)


def build(force: bool = False, verbose: bool = False, debug: bool = False, trace_only: bool = False) -> str:
    """debug=True builds libcfdetr_dbg.so with -DCFD_HANG_CHECK -DCFD_TRACE (barrier waits trap with a
    message instead of hanging); trace_only=True builds it with -DCFD_TRACE alone (release barrier
    waits, so pipeline traces keep release timing).  Load it with CFD_LIB_DEBUG=1."""
    debug = debug or trace_only
    out = LIB_DBG if debug else LIB
    if not force and os.path.exists(out) and os.path.getmtime(out) >= _newest_src_mtime():
        return out
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    tmp = out + ".tmp"
    extra = (["-DCFD_TRACE"] if trace_only else ["-DCFD_HANG_CHECK", "-DCFD_TRACE"]) if debug else []
    # extra defines for trace experiments, e.g. CFD_TRACE_DEFS="-DCFD_TRACE_MMA_PRE" (debug library only)
    extra += os.environ.get("CFD_TRACE_DEFS", "").split() if debug else []
    cmd = [nvcc(), *NVCC_FLAGS, *extra, "-shared", "-o", tmp, *srcs, "-lcudart_static", "-ldl", "-lrt", "-lpthread"]
    r = subprocess.run(cmd, cwd=CSRC, capture_output=True, text=True)
    log = os.path.join(HERE, "build_dbg.log" if debug else "build.log")
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        sys.stderr.write(r.stderr[-8000:])
        raise RuntimeError(f"nvcc failed (see {log})")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(tmp, out)
    return out


def build_variant(name: str, defines: list[str]) -> str:
    """A/B timing build: libcfdetr_<name>.so with extra -D defines (release otherwise); load it
    with CFD_LIB_VARIANT=<name>."""
    out = os.path.join(HERE, f"libcfdetr_{name}.so")
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    cmd = [nvcc(), *NVCC_FLAGS, *defines, "-shared", "-o", out, *srcs, "-lcudart_static", "-ldl", "-lrt", "-lpthread"]
    r = subprocess.run(cmd, cwd=CSRC, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stderr[-8000:])
        raise RuntimeError(f"nvcc failed for variant {name}")
    return out


if __name__ == "__main__":
    if "--variant" in sys.argv:  # python build.py --variant NAME -DX=1 ...
        i = sys.argv.index("--variant")
        print(build_variant(sys.argv[i + 1], [a for a in sys.argv[i + 2:] if a.startswith("-D")]))
        sys.exit(0)
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, debug="--debug" in sys.argv,
                trace_only="--trace" in sys.argv))
