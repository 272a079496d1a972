"""Loader for the in-tree C-ABI library ``_build/libfs_sampler.so``.

There is no CPU fallback: if the library or a CUDA device is missing, every
sampling entry point raises :class:`EngineUnavailable`.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading
from pathlib import Path

from ._abi import FS_ABI_VERSION, FsProgDesc, FsSampleOut, FsTraceIn, FsTraceOut

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "_build" / "libfs_sampler.so"
CSRC = PKG / "csrc"
INCLUDE = PKG.parent / "include"

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "--shared", "-Xcompiler", "-fPIC"]


class EngineUnavailable(RuntimeError):
    pass


_lock = threading.Lock()
_lib = None


def sources() -> list[Path]:
    return (sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.h"))
            + [INCLUDE / "fs_sampler.h"])


def build(force: bool = False, verbose: bool = False) -> Path:
    """nvcc-compile the engine for sm_100a into the package tree."""
    srcs = sources()
    newest = max(p.stat().st_mtime for p in srcs)
    if not force and LIB_PATH.exists() and LIB_PATH.stat().st_mtime >= newest:
        return LIB_PATH
    LIB_PATH.parent.mkdir(exist_ok=True)
    nvcc = os.environ.get("NVCC", "nvcc")
    if not Path(nvcc).exists():
        for cand in ("/usr/local/cuda/bin/nvcc",):
            if Path(cand).exists():
                nvcc = cand
    tmp = LIB_PATH.with_suffix(".so.tmp")
    cmd = [nvcc, *NVCC_FLAGS, "-Xptxas", "-v", "-I", str(INCLUDE), "-o", str(tmp), str(CSRC / "fs_sampler.cu")]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed:\n{res.stderr}")
    if verbose:
        print(res.stderr)
    (PKG / "_build" / "ptxas.log").write_text(res.stderr)
    # the segment-kernel headers are compiled per program at run time (NVRTC): check them here with
    # hand-written stand-ins for the generated kernels (csrc/fs_seg_check.cu), cubin only
    chk = PKG / "_build" / "fs_seg_check.cubin"
    cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-cubin",
           "-I", str(INCLUDE), "-o", str(chk), str(CSRC / "fs_seg_check.cu")]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed on the segment-kernel headers:\n{res.stderr}")
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


def lib():
    """The loaded C-ABI library (raises EngineUnavailable if it cannot be loaded)."""
    global _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise EngineUnavailable(
                    f"{LIB_PATH} is missing: run __graft_entry__.build() (nvcc, sm_100a)")
            try:
                L = C.CDLL(str(LIB_PATH))
            except OSError as exc:
                raise EngineUnavailable(f"cannot load {LIB_PATH}: {exc}") from exc
            L.fs_abi_version.restype = C.c_int
            L.fs_last_error.restype = C.c_char_p
            L.fs_program_create.restype = C.c_int
            L.fs_program_create.argtypes = [C.POINTER(FsProgDesc), C.POINTER(C.c_void_p)]
            L.fs_program_destroy.restype = None
            L.fs_program_destroy.argtypes = [C.c_void_p]
            L.fs_program_engine.restype = C.c_int
            L.fs_program_engine.argtypes = [C.c_void_p, C.c_uint32]
            L.fs_sample.restype = C.c_int
            L.fs_sample.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint32,
                                    C.POINTER(FsTraceIn), C.POINTER(FsSampleOut),
                                    C.POINTER(FsTraceOut), C.c_void_p]
            L.fs_sample_host.restype = C.c_int
            L.fs_sample_host.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint32,
                                         C.POINTER(FsTraceIn), C.POINTER(FsSampleOut),
                                         C.POINTER(FsTraceOut)]
            L.fs_accumulate.restype = C.c_int
            L.fs_accumulate.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint32,
                                        C.c_void_p, C.c_void_p]
            L.fs_format.restype = C.c_int
            L.fs_format.argtypes = [C.c_void_p, C.POINTER(FsSampleOut), C.c_uint64, C.c_int, C.c_int,
                                    C.c_uint64, C.c_char_p, C.c_void_p, C.c_uint64,
                                    C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.c_void_p]
            L.fs_format_bound.restype = C.c_uint64
            L.fs_format_bound.argtypes = [C.c_void_p, C.c_uint64, C.c_int, C.c_uint64, C.c_char_p]
            L.fs_stratum_weight.restype = C.c_int
            L.fs_stratum_weight.argtypes = [C.c_void_p, C.c_uint32, C.POINTER(C.c_double)]
            L.fs_sample_stratum.restype = C.c_int
            L.fs_sample_stratum.argtypes = [C.c_void_p, C.c_uint32, C.c_uint64, C.c_uint64, C.c_uint64,
                                            C.c_uint32, C.POINTER(FsSampleOut), C.c_void_p]
            L.fs_sample_stratum_host.restype = C.c_int
            L.fs_sample_stratum_host.argtypes = [C.c_void_p, C.c_uint32, C.c_uint64, C.c_uint64, C.c_uint64,
                                                 C.c_uint32, C.POINTER(FsSampleOut)]
            L.fs_accumulate_stratum.restype = C.c_int
            L.fs_accumulate_stratum.argtypes = [C.c_void_p, C.c_uint32, C.c_uint64, C.c_uint64, C.c_uint64,
                                                C.c_uint32, C.c_void_p, C.c_void_p]
            L.fs_probe.restype = C.c_int
            L.fs_probe.argtypes = [C.c_void_p, C.c_int32, C.c_uint64, C.c_uint64, C.c_int32,
                                   C.POINTER(C.c_double), C.c_void_p]
            if L.fs_abi_version() != FS_ABI_VERSION:
                raise EngineUnavailable("ABI version mismatch")
            _lib = L
    return _lib


def last_error() -> str:
    return (lib().fs_last_error() or b"").decode()
