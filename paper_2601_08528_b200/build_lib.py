"""Compile libsvf.so (sm_100a) in-tree with nvcc.  Used by __graft_entry__.build() and the tests' session setup."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libsvf.so")
SOURCES = ["index.cu", "search.cu", "search_d0.cu", "search_d24.cu", "search_d32.cu", "search_d50.cu", "link.cu",
           "knn.cu", "knn_tc.cu", "repair.cu"]
HEADERS = ["common.cuh", "kernels.h", "search_impl.cuh", "search_lp.cuh", os.path.join("..", "..", "include", "svf.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
         "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"] + os.environ.get("SVF_NVCC_EXTRA", "").split()


def _stale(out: str = OUT) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS] + [os.path.abspath(__file__)]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, out: str = OUT, extra: tuple = ()) -> str:
    """Compile into `out`; `extra` nvcc flags (e.g. -D knobs) build a tuning variant in its own object dir."""
    if not force and not _stale(out):
        return out
    objdir = os.path.join(HERE, "build" + ("" if out == OUT else "_" + os.path.basename(out).replace(".so", "")))
    os.makedirs(objdir, exist_ok=True)
    procs, objs = [], []
    flagfile = os.path.join(objdir, "flags.txt")
    flags_same = os.path.exists(flagfile) and open(flagfile).read() == " ".join(FLAGS + list(extra))
    def hdr_t(src):  # search_impl.cuh is included by the search TUs only
        return max(os.path.getmtime(os.path.join(CSRC, h)) for h in HEADERS
                   if src.startswith("search") or h not in ("search_impl.cuh", "search_lp.cuh"))

    for s in SOURCES:
        obj = os.path.join(objdir, s.replace(".cu", ".o"))
        objs.append(obj)
        if (not force and flags_same and os.path.exists(obj)
                and os.path.getmtime(obj) > max(hdr_t(s), os.path.getmtime(os.path.join(CSRC, s)))):
            continue                                  # object newer than its source and every header
        cmd = [NVCC, *FLAGS, *extra, "-c", os.path.join(CSRC, s), "-o", obj]
        if verbose:
            cmd += ["-Xptxas", "-v"]
        procs.append((s, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
    failed = []
    for s, p in procs:
        log, _ = p.communicate()
        if p.returncode != 0 or verbose:
            sys.stderr.write(log)
        if p.returncode != 0:
            failed.append(s)
    if failed:
        raise RuntimeError(f"nvcc failed for {failed}")
    open(flagfile, "w").write(" ".join(FLAGS + list(extra)))
    tmp = out + ".tmp"
    subprocess.check_call([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs])
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
