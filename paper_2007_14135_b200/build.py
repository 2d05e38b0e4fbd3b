"""Build libdoa.so (sm_100a) in-tree with nvcc.  Used by __graft_entry__.build() and the tests."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libdoa.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-shared", "-cudart", "static",
         "-Xptxas", "-v", "--expt-relaxed-constexpr"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def headers():
    return sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + [os.path.join(HERE, "..", "include", "doa.h")]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in sources() + headers())


def build(force: bool = False, verbose: bool = False, out: str = LIB, defines=()) -> str:
    """Compile every csrc/*.cu to an object in parallel (nvcc -c), then link libdoa.so."""
    if out == LIB and not force and not stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    tmp = out + ".tmp"
    objdir = tmp + ".objs"
    os.makedirs(objdir, exist_ok=True)
    comp = [f for f in FLAGS if f not in ("-shared", "-cudart", "static")]
    comp += os.environ.get("DOA_NVCC_EXTRA", "").split()      # tuning builds only (A/B variants)
    defs = [f"-D{d}" for d in defines]

    def one(src):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        r = subprocess.run([NVCC, *ARCH, *comp, *defs, "-c", "-o", obj, src], capture_output=True, text=True)
        return src, obj, r

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        res = list(ex.map(one, sources()))
    report = "".join(r.stdout + r.stderr for _, _, r in res)
    bad = [src for src, _, r in res if r.returncode != 0]
    if bad:
        sys.stderr.write(report)
        raise RuntimeError(f"nvcc failed building libdoa.so: {bad}")
    r = subprocess.run([NVCC, *ARCH, "-shared", "-cudart", "static", "-Xcompiler", "-fPIC", "-o", tmp,
                        *[o for _, o, _ in res]], capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed linking libdoa.so")
    if out == LIB:
        with open(os.path.join(HERE, "ptxas_report.txt"), "w") as fh:
            fh.write(report)
    if verbose:
        sys.stderr.write(report)
    os.replace(tmp, out)
    for _, o, _ in res:
        os.remove(o)
    os.rmdir(objdir)
    return out


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    outs = [a[6:] for a in sys.argv[1:] if a.startswith("--out=")]
    print(build(force="--force" in sys.argv, verbose=True, out=outs[0] if outs else LIB, defines=defs))
