"""Build libadaptis.so in-tree with nvcc for sm_100a (no JIT, no torch extension)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libadaptis.so")
# one translation unit per policy for the segment kernels, compiled in parallel
SOURCES = ["adaptis_seqg.cu", "adaptis_fixed.cu", "adaptis_inst_greedy.cu", "adaptis_inst_zb.cu", "adaptis_inst_onef1b.cu", "adaptis_inst_list.cu",
           "adaptis_inst_gpipe.cu", "adaptis_host.cu", "adaptis_kernels.cu", "adaptis_executor.cu",
           "adaptis_contend.cu"]
HEADERS = ["adaptis_internal.h", "adaptis_decode.cuh", "adaptis_seg.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden", "-Xptxas", "-v",
         "--expt-relaxed-constexpr"]


def _inputs():
    root = os.path.dirname(HERE)
    return ([os.path.join(CSRC, s) for s in SOURCES + HEADERS] +
            [os.path.join(root, "include", "adaptis.h"), __file__])


FLAG_VARS = ("ADAPTIS_GREEDY_MINB", "ADAPTIS_GREEDY_V4_MINB", "ADAPTIS_FIXED_V4_MINB", "ADAPTIS_GREEDY_COMMITS",
             "ADAPTIS_DEBUG", "ADAPTIS_KRUN", "ADAPTIS_GREEDY_ALWAYS_DECIDE", "ADAPTIS_TSTAR_REDUX",
             "ADAPTIS_SEQG_K",
             "ADAPTIS_ZB_WFILL_ONE")
STAMP = LIB + ".flags"  # the -D flags the library was built with


def _extra_flags():
    return ["-D%s=%s" % (k, os.environ[k]) for k in FLAG_VARS if os.environ.get(k)]


def build(force: bool = False, verbose: bool = False) -> str:
    extra = _extra_flags()
    stamp = " ".join(extra)
    old_stamp = open(STAMP).read() if os.path.exists(STAMP) else ""
    # stale when a source is newer than the library or the -D flags changed
    # (an A/B experiment must never measure the same binary twice)
    stale = (not os.path.exists(LIB) or max(os.path.getmtime(f) for f in _inputs()) > os.path.getmtime(LIB)
             or (os.path.exists(STAMP) or extra) and old_stamp != stamp)
    if not (force or stale):
        return LIB
    inc = ["-I", os.path.join(os.path.dirname(HERE), "include")]
    objdir = os.path.join(CSRC, "obj")
    os.makedirs(objdir, exist_ok=True)

    def compile_one(src):
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        r = subprocess.run([NVCC, *FLAGS, *extra, *inc, "-c", os.path.join(CSRC, src), "-o", obj],
                           capture_output=True, text=True)
        return obj, r

    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 1)) as ex:
        results = list(ex.map(compile_one, SOURCES))
    log_text = "".join(r.stdout + r.stderr for _, r in results)
    r = None
    if all(r_.returncode == 0 for _, r_ in results):
        r = subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                            *[o for o, _ in results], "-o", LIB + ".tmp"], capture_output=True, text=True)
        log_text += r.stdout + r.stderr
    log = os.path.join(CSRC, "ptxas.log")
    with open(log, "w") as f:
        f.write(log_text)
    if r is None or r.returncode != 0:
        sys.stderr.write(log_text[-8000:])
        raise RuntimeError("nvcc failed building libadaptis.so (see %s)" % log)
    os.replace(LIB + ".tmp", LIB)
    with open(STAMP, "w") as f:
        f.write(stamp)
    if verbose:
        print(log_text[-4000:])
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
