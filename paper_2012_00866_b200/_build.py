"""Builds libhusky.so in-tree with nvcc for sm_100a (B200) only."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libhusky.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_paths():
    """(include dir, lib dir) of the NCCL that torch ships (nvidia-nccl wheel)."""
    try:
        import nvidia.nccl as m  # noqa: F401
        base = os.path.dirname(m.__file__) if getattr(m, "__file__", None) else list(m.__path__)[0]
    except Exception:  # pragma: no cover
        base = os.path.join(sys.prefix, "lib", f"python{sys.version_info.major}.{sys.version_info.minor}",
                            "site-packages", "nvidia", "nccl")
    return os.path.join(base, "include"), os.path.join(base, "lib")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))
    deps.append(os.path.join(ROOT, "include", "husky.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str | None = None) -> str:
    """out: another output path (lab A/B builds with HUSKY_NVCC_DEFS)."""
    if out is not None:
        return _build_to(out, verbose)
    if not force and not _stale():
        return LIB
    return _build_to(LIB, verbose)


def _build_to(lib_path: str, verbose: bool) -> str:
    inc, libdir = nccl_paths()
    objdir = os.path.join(HERE, "build") if lib_path == LIB else lib_path + ".objs"
    os.makedirs(objdir, exist_ok=True)
    common = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", *ARCH, f"-I{inc}",
              "-DNDEBUG", "--expt-relaxed-constexpr"]
    # instrumented builds (per-tile phase timestamps): HUSKY_NVCC_DEFS="-DHUSKY_TIMING"
    common += os.environ.get("HUSKY_NVCC_DEFS", "").split()
    objs = []
    procs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [NVCC, *common, "-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd))
        procs.append((subprocess.Popen(cmd), cmd))
        objs.append(obj)
    for p, cmd in procs:
        if p.wait() != 0:
            raise RuntimeError("nvcc failed: " + " ".join(cmd))
    tmp = lib_path + f".tmp{os.getpid()}"
    link = [NVCC, "-shared", *ARCH, "-o", tmp, *objs, f"-L{libdir}", "-l:libnccl.so.2",
            f"-Xlinker", f"-rpath={libdir}", "-lcudart"]
    if verbose:
        print(" ".join(link))
    subprocess.check_call(link)
    os.replace(tmp, lib_path)
    return lib_path


def build_cub_bar(force: bool = False) -> str:
    """tools/libcubbar.so: cub::DeviceRadixSort::SortPairs, the stage-2 library bar
    bench.py reports beside the hand-written onesweep (bench infrastructure)."""
    src = os.path.join(ROOT, "tools", "cub_bar.cu")
    out = os.path.join(ROOT, "tools", "libcubbar.so")
    if force or not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(src):
        tmp = out + f".tmp{os.getpid()}"
        subprocess.check_call([NVCC, "-O3", "-std=c++17", "-shared", "-Xcompiler", "-fPIC", *ARCH, "-o", tmp, src])
        os.replace(tmp, out)
    return out


if __name__ == "__main__":
    # python _build.py [--force] [--out PATH]   (HUSKY_NVCC_DEFS="-D..." for lab variants)
    o = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else None
    print(build(force="--force" in sys.argv, verbose=True, out=o))
