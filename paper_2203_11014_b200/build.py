"""Build libdhen.so in-tree with nvcc for sm_100a (no torch extension machinery).

    python -m paper_2203_11014_b200.build [--force] [--watchdog]

Objects go to paper_2203_11014_b200/build/, the library to
paper_2203_11014_b200/libdhen.so (git-ignored, travels to the GPU box).
--watchdog builds the debug variant libdhen_wd.so (objects in build_wd/):
every mbarrier wait is bounded and reports its call site before trapping
(common.cuh); load it with binding.load(binding.WD_LIB_PATH).
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libdhen.so")
WD_LIB = os.path.join(HERE, "libdhen_wd.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dir() -> str:
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in list(spec.submodule_search_locations or []):
        d = os.path.join(base, "nccl")
        if os.path.exists(os.path.join(d, "include", "nccl.h")):
            return d
    raise RuntimeError("nccl headers not found under the nvidia python package")


def _flags():
    nd = nccl_dir()
    return ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
                   "-I", os.path.join(nd, "include"), "-I", os.path.join(ROOT, "include"),
                   "-Xptxas", "-warn-spills"], nd


def _deps_newer(obj: str, src: str) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    hdrs = glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        glob.glob(os.path.join(ROOT, "include", "*.h"))
    return any(os.path.getmtime(p) > t for p in [src] + hdrs)


def build(force: bool = False, verbose: bool = False, watchdog: bool = False) -> str:
    bdir, lib_out = (BUILD + "_wd", WD_LIB) if watchdog else (BUILD, LIB)
    os.makedirs(bdir, exist_ok=True)
    flags, nd = _flags()
    if watchdog:
        flags = flags + ["-DDHEN_WATCHDOG=1"]
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    jobs = []
    for s in srcs:
        o = os.path.join(bdir, os.path.basename(s) + ".o")
        if force or _deps_newer(o, s):
            jobs.append((s, o))

    def comp(job):
        s, o = job
        cmd = [NVCC] + flags + ["-c", s, "-o", o]
        r = subprocess.run(cmd, capture_output=True, text=True)
        return s, r

    failed = []
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        for s, r in ex.map(comp, jobs):
            out = (r.stdout + r.stderr).strip()
            if r.returncode != 0:
                failed.append(f"{os.path.basename(s)}:\n{out}")
            elif verbose and out:
                print(f"{os.path.basename(s)}: {out}")
    if failed:
        raise RuntimeError("nvcc failed:\n" + "\n".join(failed))
    objs = [os.path.join(bdir, os.path.basename(s) + ".o") for s in srcs]
    if force or jobs or not os.path.exists(lib_out):
        lib = os.path.join(nd, "lib")
        cmd = [NVCC] + ARCH + ["-shared", "-o", lib_out] + objs + \
            ["-L", lib, "-l:libnccl.so.2", "-Xlinker", f"-rpath={lib}", "-lcuda"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("link failed:\n" + r.stdout + r.stderr)
    return lib_out


def build_probe(n: int) -> str:
    """Race-probe test build libdhen_probe<n>.so (tests/test_gpu_attn.py): attn_tc.cu recompiled with bounded
    mbarrier waits (2 s) and delay injection (DHEN_RACE_PROBE = n: 1 current protocol, 2 round 1's dh = 64
    backward protocol), linked with the default build's other objects."""
    build()
    flags, nd = _flags()
    pdir = BUILD + f"_probe{n}"
    os.makedirs(pdir, exist_ok=True)
    src = os.path.join(CSRC, "attn_tc.cu")
    obj = os.path.join(pdir, "attn_tc.cu.o")
    out = os.path.join(HERE, f"libdhen_probe{n}.so")
    if _deps_newer(obj, src) or not os.path.exists(out):
        cmd = [NVCC] + flags + ["-DDHEN_WATCHDOG=1", "-DDHEN_WATCHDOG_NS=2000000000ull", f"-DDHEN_RACE_PROBE={n}",
                                "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + r.stdout + r.stderr)
        objs = [obj] + [os.path.join(BUILD, os.path.basename(x) + ".o") for x in sorted(glob.glob(os.path.join(CSRC, "*.cu")))
                        if os.path.basename(x) != "attn_tc.cu"]
        lib = os.path.join(nd, "lib")
        r = subprocess.run([NVCC] + ARCH + ["-shared", "-o", out] + objs +
                           ["-L", lib, "-l:libnccl.so.2", "-Xlinker", f"-rpath={lib}", "-lcuda"], capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("link failed:\n" + r.stdout + r.stderr)
    return out


if __name__ == "__main__":
    if "--probe" in sys.argv:
        print(build_probe(int(sys.argv[sys.argv.index("--probe") + 1])))
    else:
        print(build(force="--force" in sys.argv, verbose=True, watchdog="--watchdog" in sys.argv))
