"""In-tree build of libmoeplan_b200.so (host planner C++ + sm_100a CUDA + C ABI).

No torch extension machinery: g++ for the host planner (-ffp-contract=off, the
planner's doubles must round exactly like the reference's), nvcc with
``-gencode arch=compute_100a,code=sm_100a -lineinfo`` for the kernels and the
runtime, linked against the NCCL 2.28 that torch ships (one NCCL per process).
The .so lands in ``paper_2602_11686_b200/lib/`` so it travels to the GPU box with
the repo snapshot.  Incremental: objects are rebuilt when a source or any header
under csrc/ or include/ is newer.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
import sysconfig
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIBDIR = PKG / "lib"
OBJDIR = LIBDIR / "obj"
LIBNAME = "libmoeplan_b200.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _site() -> Path:
    return Path(sysconfig.get_paths()["purelib"])


def _json_dir() -> Path:
    return _site() / "include" / "cudnn_frontend" / "thirdparty" / "nlohmann"


def _nccl_dir() -> Path:
    return _site() / "nvidia" / "nccl"


def _cuda_home() -> Path:
    return Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))


def lib_path() -> Path:
    # FSEP_LIB_NAME selects a dev variant (e.g. a -DFSEP_GEMM_STALLS build, with its own objects)
    return LIBDIR / os.environ.get("FSEP_LIB_NAME", LIBNAME)


def _objdir() -> Path:
    v = os.environ.get("FSEP_LIB_NAME")
    return OBJDIR if not v else LIBDIR / ("obj_" + v.replace(".so", ""))


def _headers_mtime() -> float:
    newest = 0.0
    for d in (CSRC, ROOT / "include"):
        for p in d.rglob("*"):
            if p.suffix in (".h", ".hpp", ".cuh"):
                newest = max(newest, p.stat().st_mtime)
    return newest


def _sources():
    host = sorted((CSRC / "host").glob("*.cpp"))
    cuda = sorted((CSRC / "kernels").glob("*.cu")) + sorted((CSRC / "runtime").glob("*.cu"))
    return host, cuda


def _run(cmd):
    r = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
    if r.returncode != 0:
        raise RuntimeError("build failed:\n" + " ".join(map(str, cmd)) + "\n" + r.stdout)
    return r.stdout


def build(verbose: bool = False, force: bool = False, jobs: int | None = None) -> Path:
    objdir = _objdir()
    objdir.mkdir(parents=True, exist_ok=True)
    host, cuda = _sources()
    hdr_t = _headers_mtime()
    inc = ["-I", str(ROOT / "include"), "-I", str(CSRC), "-I", str(_json_dir()),
           "-I", str(_nccl_dir() / "include")]
    cxx = ["g++", "-std=c++20", "-O2", "-fPIC", "-ffp-contract=off", "-Wall",
           "-Wno-unused-function", "-isystem", str(_cuda_home() / "include")] + inc
    nvcc = [str(_cuda_home() / "bin" / "nvcc"), "-std=c++20", "-O3", "-lineinfo", *ARCH,
            "-Xcompiler", "-fPIC,-ffp-contract=off", "--expt-relaxed-constexpr",
            "-Xptxas", "-v" if verbose else "-O3"] + os.environ.get("FSEP_NVCC_EXTRA", "").split() + inc
    jobs_ = []
    objs = []
    for src in host + cuda:
        obj = objdir / (src.stem + (".cu.o" if src.suffix == ".cu" else ".o"))
        objs.append(obj)
        if not force and obj.exists() and obj.stat().st_mtime >= max(src.stat().st_mtime, hdr_t):
            continue
        cmd = (nvcc if src.suffix == ".cu" else cxx) + ["-c", str(src), "-o", str(obj)]
        jobs_.append(cmd)
    with cf.ThreadPoolExecutor(max_workers=jobs or os.cpu_count() or 4) as ex:
        for out in ex.map(_run, jobs_):
            if verbose and out.strip():
                print(out, file=sys.stderr)
    lib = lib_path()
    if jobs_ or not lib.exists() or force:
        nccl_lib = _nccl_dir() / "lib"
        link = ["g++", "-shared", "-o", str(lib) + ".tmp", *map(str, objs),
                "-L", str(_cuda_home() / "lib64"), "-lcudart",
                "-L", str(nccl_lib), "-l:libnccl.so.2",
                f"-Wl,-rpath,{nccl_lib}", f"-Wl,-rpath,{_cuda_home() / 'lib64'}",
                "-Wl,-Bsymbolic", "-Wl,--no-undefined"]
        _run(link)
        shutil.move(str(lib) + ".tmp", lib)
    return lib


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
