"""Builds the in-tree CUDA library lib/libfastclip_b200.so for sm_100a with nvcc.

The kernels are hand-written tcgen05/TMA code (csrc/), compiled with
`-gencode arch=compute_100a,code=sm_100a -lineinfo`; the host runtime links NCCL from the
same wheel torch uses (nvidia-nccl-cu12), so one libnccl is loaded per process.
"""
from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIBDIR, "libfastclip_b200.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in (spec.submodule_search_locations or []) if spec else []:
        inc, lib = os.path.join(base, "nccl", "include"), os.path.join(base, "nccl", "lib")
        if os.path.exists(os.path.join(lib, "libnccl.so.2")):
            return inc, lib
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def flavor() -> str:
    return "profile" if os.environ.get("FC_PROFILE") == "1" else "release"


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    stamp = LIB + ".flavor"   # a profiling build never passes for the release one (or back)
    if not os.path.exists(stamp) or open(stamp).read().strip() != flavor():
        return False
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [
        os.path.join(HERE, "..", "include", "fastclip_b200.h")]
    return all(os.path.getmtime(p) <= t for p in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    inc, lib = nccl_dirs()
    os.makedirs(LIBDIR, exist_ok=True)
    objs, procs = [], []
    for src in sources():
        obj = os.path.join(LIBDIR, os.path.basename(src) + ".o")
        cmd = [nvcc, *ARCH, "-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-I", inc,
               "-c", src, "-o", obj]
        if os.environ.get("FC_PROFILE") == "1":   # profiling build: globaltimer / cycle stamps compiled in
            cmd.insert(1, "-DFC_PROFILE")
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        procs.append((subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT), src))
        objs.append(obj)
    for p, src in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{out.decode()}")
        if verbose:
            print(out.decode())
    tmp = LIB + ".tmp"
    link = [nvcc, *ARCH, "-shared", "-o", tmp, *objs, "-L", lib, "-l:libnccl.so.2",
            "-Xlinker", f"-rpath,{lib}"]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    with open(LIB + ".flavor", "w") as fh:
        fh.write(flavor() + "\n")
    for o in objs:
        os.remove(o)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
