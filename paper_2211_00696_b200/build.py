"""In-tree build of libpq_b200.so (sm_100a) — called by __graft_entry__.build().

nvcc compiles the kernels for `-gencode arch=compute_100a,code=sm_100a` only; g++ compiles the
host engine (C++20, no -ffast-math / -mfma so the estimator rounds like the reference).  The CUDA
runtime is linked statically and its symbols hidden, so the library coexists with torch's cudart.
Objects are rebuilt only when a source or header is newer.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = PKG / "_build"
LIB = PKG / "libpq_b200.so"
CLI = PKG / "phiquad_cli"  # the reference CLI's wire format on this engine (cli/phiquad_cli.cpp)
CUDA = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

CU_SOURCES = ["gemm_nk.cu", "gemm_kk.cu", "slab12.cu", "kernels.cu"]
CPP_SOURCES = ["estimator.cpp", "engine.cpp", "etd.cpp", "capi.cpp", "dist.cpp"]


def _headers() -> list[Path]:
    return list(CSRC.glob("*.hpp")) + list(CSRC.glob("*.cuh")) + list((ROOT / "include").glob("*.h"))


def _stale(src: Path, obj: Path) -> bool:
    if not obj.exists():
        return True
    t = obj.stat().st_mtime
    return src.stat().st_mtime > t or any(h.stat().st_mtime > t for h in _headers())


def _nvcc() -> str:
    p = shutil.which("nvcc") or str(CUDA / "bin" / "nvcc")
    return p


def _cmd_cu(src: Path, obj: Path) -> list[str]:
    return [_nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-fvisibility=hidden",
            "-I", str(ROOT / "include"), "-I", str(CSRC), "-c", str(src), "-o", str(obj)]


def _cmd_cpp(src: Path, obj: Path) -> list[str]:
    cxx = os.environ.get("CXX", "g++")
    return [cxx, "-std=c++20", "-O3", "-fPIC", "-fvisibility=hidden", "-Wall", "-Wno-unused-function",
            "-I", str(ROOT / "include"), "-I", str(CSRC), "-I", str(CUDA / "include"), "-c", str(src), "-o", str(obj)]


def build(verbose: bool = False) -> Path:
    OBJ.mkdir(exist_ok=True)
    jobs = []
    for name in CU_SOURCES:
        src, obj = CSRC / name, OBJ / (name + ".o")
        if _stale(src, obj):
            jobs.append(_cmd_cu(src, obj))
    for name in CPP_SOURCES:
        src, obj = CSRC / name, OBJ / (name + ".o")
        if _stale(src, obj):
            jobs.append(_cmd_cpp(src, obj))

    def run(cmd: list[str]) -> None:
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")

    with cf.ThreadPoolExecutor(max_workers=max(1, os.cpu_count() or 1)) as ex:
        list(ex.map(run, jobs))
    objs = [str(OBJ / (n + ".o")) for n in CU_SOURCES + CPP_SOURCES]
    if jobs or not LIB.exists() or any(Path(o).stat().st_mtime > LIB.stat().st_mtime for o in objs):
        link = [os.environ.get("CXX", "g++"), "-shared", "-o", str(LIB), *objs,
                "-L", str(CUDA / "lib64"), "-lcudart_static", "-ldl", "-lrt", "-lpthread",
                "-Wl,--exclude-libs,ALL", "-Wl,-soname,libpq_b200.so"]
        run(link)
    cli_src = PKG / "cli" / "phiquad_cli.cpp"
    headers = list((ROOT / "include" / "phiquad").glob("*.hpp"))
    if not CLI.exists() or any(p.stat().st_mtime > CLI.stat().st_mtime for p in [cli_src, LIB, *headers]):
        run([os.environ.get("CXX", "g++"), "-std=c++20", "-O2", "-pthread", "-I", str(ROOT / "include"), str(cli_src),
             "-L", str(PKG), "-lpq_b200", "-Wl,-rpath,$ORIGIN", "-o", str(CLI)])
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
