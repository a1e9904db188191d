"""Build libadaptis.so in-tree with nvcc for sm_100a (no JIT, no torch extension)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libadaptis.so")
SOURCES = ["adaptis_host.cu", "adaptis_kernels.cu"]
HEADERS = ["adaptis_internal.h", "adaptis_decode.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden", "-Xptxas", "-v",
         "--expt-relaxed-constexpr", "-shared"]


def _inputs():
    root = os.path.dirname(HERE)
    return ([os.path.join(CSRC, s) for s in SOURCES + HEADERS] +
            [os.path.join(root, "include", "adaptis.h"), __file__])


def build(force: bool = False, verbose: bool = False) -> str:
    stale = not os.path.exists(LIB) or max(os.path.getmtime(f) for f in _inputs()) > os.path.getmtime(LIB)
    if not (force or stale):
        return LIB
    extra = ["-D%s=%s" % (k, os.environ[k]) for k in ("ADAPTIS_GREEDY_MINB", "ADAPTIS_GREEDY_V4_MINB", "ADAPTIS_FIXED_V4_MINB", "ADAPTIS_GREEDY_COMMITS", "ADAPTIS_DEBUG", "ADAPTIS_KRUN", "ADAPTIS_GREEDY_ALWAYS_DECIDE") if os.environ.get(k)]
    cmd = [NVCC, *FLAGS, *extra, "-I", os.path.join(os.path.dirname(HERE), "include"),
           *[os.path.join(CSRC, s) for s in SOURCES], "-o", LIB + ".tmp"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(CSRC, "ptxas.log")
    with open(log, "w") as f:
        f.write(r.stdout + r.stderr)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libadaptis.so (see %s)" % log)
    os.replace(LIB + ".tmp", LIB)
    if verbose:
        print(r.stderr[-4000:])
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
