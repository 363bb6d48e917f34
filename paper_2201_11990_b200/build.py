"""In-tree build of the native library `libmtnlg.so` (sm_100a CUDA kernels + C++ host runtime).

Every .cu under csrc/ is compiled with nvcc for sm_100a only; every .cpp with g++ -std=c++20.
The result lands next to this file so it travels to the GPU box with the repo snapshot
(gpurun copies built .so files; a JIT cache under ~/.cache would not).
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
# MT_NVCC_DEFINES (A/B builds of compile-time variants, e.g. "-DMT_GEMM_EPI_BUFS=4"): separate object dir
_VARIANT = os.environ.get("MT_NVCC_DEFINES", "").split()
OBJ = ROOT / "build" / ("obj" if not _VARIANT else "obj_" + "_".join(d.lstrip("-D").replace("=", "") for d in _VARIANT))
LIB = PKG / "libmtnlg.so"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _nccl_root() -> Path | None:
    """NCCL >= 2.28 (device API: symmetric windows, multimem pointers) — the copy shipped with torch."""
    try:
        import nvidia.nccl  # namespace package of the nvidia-nccl wheel
        for p in nvidia.nccl.__path__:
            if (Path(p) / "include" / "nccl_device.h").exists():
                return Path(p)
    except ImportError:
        pass
    return None


NCCL = _nccl_root()
if NCCL is None:
    raise RuntimeError("NCCL >= 2.28 headers (nccl_device.h) not found: the fused TP all-reduce needs the NCCL device API")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
INCLUDES = [f"-I{ROOT / 'include'}", f"-I{CSRC}", f"-I{NCCL / 'include'}", "-I/usr/local/cuda/include"]
NVCC_FLAGS = ARCH + ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-fopenmp", "--expt-relaxed-constexpr"] + _VARIANT
CXX_FLAGS = ["-O3", "-std=c++20", "-fPIC", "-fopenmp", "-Wall", "-Wextra", "-Wno-unused-parameter"]


def _deps(src: Path) -> list[Path]:
    hdrs = list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.hpp")) + list((ROOT / "include").rglob("*.h*"))
    return [src] + hdrs


def _stale(obj: Path, src: Path) -> bool:
    if not obj.exists():
        return True
    t = obj.stat().st_mtime
    return any(d.stat().st_mtime > t for d in _deps(src))


def _run(cmd: list[str]) -> None:
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        raise RuntimeError(f"build failed: {cmd[0]} {cmd[-1]}")


def build(verbose: bool = False, jobs: int = 8) -> Path:
    OBJ.mkdir(parents=True, exist_ok=True)
    cmds, objs = [], []
    for src in sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cpp")):
        obj = OBJ / (src.name + ".o")
        objs.append(obj)
        if not _stale(obj, src):
            continue
        if src.suffix == ".cu":
            cmds.append([NVCC, *NVCC_FLAGS, *INCLUDES, "-c", str(src), "-o", str(obj)])
        else:
            cmds.append(["g++", *CXX_FLAGS, *INCLUDES, "-c", str(src), "-o", str(obj)])
    # compile in parallel
    procs = []
    for cmd in cmds:
        if verbose:
            print(" ".join(cmd))
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
        if len(procs) >= jobs:
            _drain(procs)
    _drain(procs)
    newest = max(o.stat().st_mtime for o in objs)
    # the library records which object set it was linked from, so the default build relinks after an
    # A/B variant build even when the default objects are older than the variant's library
    stamp = ROOT / "build" / "libmtnlg.variant"
    want = " ".join(_VARIANT)
    linked = stamp.read_text() if stamp.exists() else None
    if linked != want or not LIB.exists() or LIB.stat().st_mtime < newest:
        _run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", str(LIB), *map(str, objs),
              f"-L{NCCL / 'lib'}", "-l:libnccl.so.2", "-Xlinker", f"-rpath={NCCL / 'lib'}",
              "-Xcompiler", "-fopenmp", "-lgomp"])
        stamp.write_text(want)
    return LIB


def _drain(procs: list) -> None:
    err = None
    for cmd, p in procs:
        out, e = p.communicate()
        if p.returncode != 0:
            sys.stderr.write(" ".join(cmd) + "\n" + out + e)
            err = cmd
    procs.clear()
    if err:
        raise RuntimeError(f"build failed: {err[-1]}")


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
