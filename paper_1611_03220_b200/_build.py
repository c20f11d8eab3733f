"""In-tree build of the CUDA library (sm_100a) and of the CPU oracle.

`python paper_1611_03220_b200/_build.py` (or __graft_entry__.build()) compiles
every translation unit under csrc/ with nvcc for sm_100a only and links
paper_1611_03220_b200/libkrr_b200.so (rpath to the CUDA and NCCL libraries).
The .so is git-ignored but travels to the GPU box with the gpurun snapshot.
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
BUILD = PKG / "_obj"
LIB = PKG / "libkrr_b200.so"
DIAG_SRC = PKG / "diag"
DIAG_LIB = PKG / "libkrr_diag.so"
ORACLE_DIR = ROOT / "oracle"
CUDA_HOME = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))
NVCC = str(CUDA_HOME / "bin" / "nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + [
    "-O3", "-lineinfo", "-std=c++20", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
    "-I", str(ROOT / "include"),
]
LINK_LIBS = [
    "-L", str(CUDA_HOME / "lib64"), "-lcublas", "-lcusolver", "-lcudart",
    "-ldl",
    "-Xlinker", "-rpath," + str(CUDA_HOME / "lib64"),
]


def _sources():
    return sorted(list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cpp")))


def _headers_mtime() -> float:
    hs = (list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.hpp")) + list((ROOT / "include").glob("*.h")) +
          list(DIAG_SRC.glob("*.cuh")))
    return max((h.stat().st_mtime for h in hs), default=0.0)


def _compile(src: Path, verbose: bool, prefix: str = "") -> Path:
    obj = BUILD / (prefix + src.name + ".o")
    hm = _headers_mtime()
    if obj.exists() and obj.stat().st_mtime >= max(src.stat().st_mtime, hm):
        return obj
    cmd = [NVCC] + NVCC_FLAGS + ["-I", str(CSRC), "-c", str(src), "-o", str(obj)]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{res.stderr}\n{res.stdout}")
    if verbose and res.stderr:
        print(res.stderr, file=sys.stderr)
    return obj


def build_lib(verbose: bool = False, force: bool = False) -> Path:
    BUILD.mkdir(exist_ok=True)
    if force:
        for o in BUILD.glob("*.o"):
            o.unlink()
    srcs = _sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), srcs))
    newest = max(o.stat().st_mtime for o in objs)
    if LIB.exists() and LIB.stat().st_mtime >= newest and not force:
        return LIB
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [NVCC] + ARCH + ["-shared", "-o", str(tmp)] + [str(o) for o in objs] + LINK_LIBS
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stderr}\n{res.stdout}")
    os.replace(tmp, LIB)
    return LIB


def build_diag(verbose: bool = False, force: bool = False) -> Path:
    """libkrr_diag.so: micro-benchmarks / probes / traces (include/krr_diag.h), linked against
    the product library; not part of the drop-in interface."""
    BUILD.mkdir(exist_ok=True)
    srcs = sorted(DIAG_SRC.glob("*.cu"))
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose, "diag_"), srcs))
    newest = max([o.stat().st_mtime for o in objs] + [LIB.stat().st_mtime])
    if DIAG_LIB.exists() and DIAG_LIB.stat().st_mtime >= newest and not force:
        return DIAG_LIB
    tmp = DIAG_LIB.with_suffix(".so.tmp")
    cmd = ([NVCC] + ARCH + ["-shared", "-o", str(tmp)] + [str(o) for o in objs] + LINK_LIBS +
           ["-L", str(PKG), "-lkrr_b200", "-Xlinker", "-rpath,$ORIGIN"])
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"diag link failed:\n{res.stderr}\n{res.stdout}")
    os.replace(tmp, DIAG_LIB)
    return DIAG_LIB


def build_examples() -> Path:
    """C++ caller of the C-ABI (examples/cpp_dropin.cpp), linked against the in-tree .so."""
    src = ROOT / "examples" / "cpp_dropin.cpp"
    out = ROOT / "examples" / "cpp_dropin"
    if out.exists() and out.stat().st_mtime >= max(src.stat().st_mtime, LIB.stat().st_mtime):
        return out
    cmd = ["g++", "-O2", "-std=c++20", "-I", str(ROOT / "include"), str(src), "-o", str(out),
           "-L", str(PKG), "-lkrr_b200", "-Wl,-rpath,$ORIGIN/../paper_1611_03220_b200"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"example build failed:\n{res.stderr}")
    return out


def build_oracle() -> Path:
    """CPU restatement used only by tests / the CPU baseline (oracle/Makefile)."""
    make = shutil.which("make")
    if make is None:
        raise RuntimeError("make not found")
    res = subprocess.run([make, "-C", str(ORACLE_DIR)], capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"oracle build failed:\n{res.stderr}\n{res.stdout}")
    return ORACLE_DIR / "liboracle.so"


def main(argv=None) -> int:
    argv = list(sys.argv[1:] if argv is None else argv)
    verbose = "-v" in argv
    force = "-f" in argv
    lib = build_lib(verbose=verbose, force=force)
    diag = build_diag(verbose=verbose, force=force)
    orc = build_oracle()
    ex = build_examples()
    print(lib)
    print(diag)
    print(orc)
    print(ex)
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
