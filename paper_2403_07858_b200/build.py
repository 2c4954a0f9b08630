"""Build the sm_100a shared library in-tree (``libbicount_b200.so``).

Plain nvcc, no torch extension machinery: the product is a C-ABI ``.so``
loaded through ctypes (``_abi.py``).  Flags: ``-gencode
arch=compute_100a,code=sm_100a -lineinfo -O3``.
"""

from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libbicount_b200.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3",
         "--expt-relaxed-constexpr"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps() -> list[str]:
    return sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + [
        os.path.join(HERE, "..", "include", "bicount_b200.h")]


def source_hash() -> str:
    """sha256 (16 hex) of every build input and the nvcc flags: the key under which ncu
    captures of this build are filed (profiles/r2/traffic.json)."""
    import hashlib

    h = hashlib.sha256(" ".join(FLAGS).encode())
    for d in sorted(deps(), key=os.path.basename):
        h.update(os.path.basename(d).encode())
        with open(d, "rb") as f:
            h.update(f.read())
    return h.hexdigest()[:16]


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(d) <= t for d in deps())


def build(force: bool = False, verbose: bool = False, extra: list[str] | None = None,
          out: str | None = None) -> str:
    lib = out or LIB
    if not force and out is None and up_to_date():
        return LIB
    # one nvcc per translation unit in parallel, then one link
    flags = [*FLAGS, *(extra or [])]
    if verbose:
        flags.insert(0, "-Xptxas=-v")
    tag = os.path.basename(lib).replace(".so", "")
    objs, procs = [], []
    for src in sources():
        obj = os.path.join(CSRC, f".{tag}.{os.path.basename(src)}.o")
        objs.append(obj)
        procs.append((src, subprocess.Popen([nvcc(), *flags, "-c", "-o", obj, src],
                                            stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                                            text=True)))
    failed = False
    for src, pr in procs:
        out_, err_ = pr.communicate()
        if pr.returncode != 0:
            failed = True
            sys.stderr.write(out_ + err_)
        elif verbose:
            sys.stderr.write(err_)
    if failed:
        raise RuntimeError("nvcc build of libbicount_b200.so failed")
    r = subprocess.run([nvcc(), *ARCH, "-shared", "-o", lib + ".tmp", *objs, "-lcudart"],
                       capture_output=True, text=True)
    for o in objs:
        if os.path.exists(o):
            os.remove(o)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link of libbicount_b200.so failed")
    os.replace(lib + ".tmp", lib)
    return lib


if __name__ == "__main__":
    if "--variant" in sys.argv:  # development variants: --variant NAME -DX=Y ...
        i = sys.argv.index("--variant")
        name, defs = sys.argv[i + 1], [a for a in sys.argv[i + 2:] if a.startswith("-D")]
        print(build(force=True, verbose="-v" in sys.argv, extra=defs,
                    out=os.path.join(HERE, f"libbicount_b200_{name}.so")))
    elif "--prof" in sys.argv:  # phase-profiling development build (BC_LIB=... to load it)
        print(build(force=True, verbose="-v" in sys.argv, extra=["-DBC_PHASE_PROF"],
                    out=os.path.join(HERE, "libbicount_b200_prof.so")))
    else:
        build(force="--force" in sys.argv, verbose="-v" in sys.argv)
        print(LIB)
