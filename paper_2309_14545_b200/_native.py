"""ctypes binding of libvmp.so (include/vmp.h) and its in-tree build.

The shared library lives next to this file and is built by ``build_native()``
(called from __graft_entry__.build()).  Loading it never needs a GPU; any
compute call on a machine without one fails loudly with RuntimeError.  There
is deliberately no fallback: if the library is missing the import of the
product API raises.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB_PATH = PKG / "libvmp.so"
INCLUDE = PKG.parent / "include"

VMP_OK = 0
VMP_EARG = -1
VMP_ECUDA = -2
VMP_ECOMPILE = -3

VMP_PRUNE = 1
VMP_NO_EARLY_EXIT = 4
VMP_NO_SPLIT = 8
VMP_FORCE_SPLIT = 32
VMP_TWO_PASS = 64
VMP_BACKWARD = 16
VMP_OVERLAPPED = 512
VMP_PDL = 1024

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo", "-O3", "-std=c++17",
    "-shared", "-Xcompiler", "-fPIC",
]

#: every symbol include/vmp.h declares (checked by the CPU tests)
EXPORTS = (
    "vmp_version", "vmp_last_error", "vmp_compile", "vmp_robot_load", "vmp_robot_destroy",
    "vmp_env_create", "vmp_env_create_at", "vmp_env_destroy", "vmp_env_bytes", "vmp_fk_rows",
    "vmp_fk_spheres",
    "vmp_validate", "vmp_validate_motions", "vmp_discretize", "vmp_sphere_hits",
    "vmp_set_device", "vmp_device_info", "vmp_motion_workspace_bytes", "vmp_pair_clear",
    "vmp_knn", "vmp_nn_distances", "vmp_debug_motion_trace", "vmp_robot_home",
    "vmp_motion_states", "vmp_bench_ffma", "vmp_validate_host", "vmp_validate_host_scratch_bytes",
    "vmp_validate_motions_host", "vmp_motions_host_scratch_bytes", "vmp_device_alloc",
    "vmp_device_free",
)
VMP_KNN_MAX_K = 32
VMP_KNN_MAX_DIM = 64


class RobotDesc(ctypes.Structure):
    _fields_ = [("dof", ctypes.c_int32), ("n_ops", ctypes.c_int32),
                ("n_markers", ctypes.c_int32), ("has_cc", ctypes.c_int32)]


def _sources() -> list[Path]:
    return [CSRC / "vmp.cu", CSRC / "vmp_device.cuh", CSRC / "vmp_abi.h", INCLUDE / "vmp.h"]


def needs_build() -> bool:
    if not LIB_PATH.exists():
        return True
    built = LIB_PATH.stat().st_mtime
    return any(src.stat().st_mtime > built for src in _sources())


def build_native(force: bool = False, verbose: bool = False) -> Path:
    """nvcc -> libvmp.so for sm_100a (cross-compiles without a GPU)."""
    if not force and not needs_build():
        return LIB_PATH
    tmp = LIB_PATH.with_suffix(".so.tmp")
    cmd = ["nvcc", *NVCC_FLAGS, f"-I{CSRC}", "-o", str(tmp), str(CSRC / "vmp.cu"),
           "-lnvrtc", "-Xlinker", "-rpath,/usr/local/cuda/lib64"]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.run(cmd, check=True, capture_output=not verbose)
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


_LIB = None


def lib() -> ctypes.CDLL:
    global _LIB
    if _LIB is not None:
        return _LIB
    if not LIB_PATH.exists():
        raise ImportError(f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; "
                          f"g.build()'` (no CPU fallback exists)")
    L = ctypes.CDLL(str(LIB_PATH))
    c_i32, c_i64, c_u32, c_dbl = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, ctypes.c_double
    vp, cp = ctypes.c_void_p, ctypes.c_char_p
    sig = {
        "vmp_version": ([], ctypes.c_int),
        "vmp_last_error": ([], cp),
        "vmp_compile": ([cp, cp, cp], ctypes.c_int),
        "vmp_robot_load": ([cp, ctypes.POINTER(RobotDesc), ctypes.POINTER(vp)], ctypes.c_int),
        "vmp_robot_destroy": ([vp], None),
        "vmp_env_create": ([vp, c_i32, vp, c_i32, vp, c_i32, ctypes.POINTER(vp)], ctypes.c_int),
        "vmp_env_create_at": ([vp, c_i32, vp, c_i32, vp, c_i32, vp, ctypes.POINTER(vp)],
                              ctypes.c_int),
        "vmp_env_destroy": ([vp], None),
        "vmp_robot_home": ([vp, vp], ctypes.c_int),
        "vmp_env_bytes": ([vp], c_i64),
        "vmp_fk_rows": ([vp, vp, c_i64, c_i64, vp, c_i64, vp], ctypes.c_int),
        "vmp_fk_spheres": ([vp, vp, c_i64, c_i64, vp, c_i64, vp], ctypes.c_int),
        "vmp_validate": ([vp, vp, vp, c_i64, c_i64, c_u32, vp, vp], ctypes.c_int),
        "vmp_validate_motions": ([vp, vp, vp, vp, c_i64, c_i64, c_dbl, c_i32, c_u32, vp, vp, vp,
                                  vp, c_i64, vp], ctypes.c_int),
        "vmp_motion_workspace_bytes": ([c_i64], c_i64),
        "vmp_discretize": ([vp, vp, c_i64, c_i32, c_i64, c_dbl, vp, vp], ctypes.c_int),
        "vmp_validate_host": ([vp, vp, vp, c_i64, c_i64, c_u32, vp, vp, c_i64, vp], ctypes.c_int),
        "vmp_validate_host_scratch_bytes": ([vp, c_i64], c_i64),
        "vmp_validate_motions_host": ([vp, vp, vp, vp, c_i64, c_i64, c_dbl, c_i32, c_u32, vp, vp, vp,
                                       vp, c_i64, vp, c_i64, vp], ctypes.c_int),
        "vmp_motions_host_scratch_bytes": ([vp, c_i64], c_i64),
        "vmp_device_alloc": ([c_i64, ctypes.POINTER(vp)], ctypes.c_int),
        "vmp_device_free": ([vp], None),
        "vmp_bench_ffma": ([c_i64, c_i32, ctypes.POINTER(c_dbl), ctypes.POINTER(c_dbl)],
                           ctypes.c_int),
        "vmp_motion_states": ([vp, vp, c_i64, c_i32, c_i64, c_dbl, c_i32, c_u32, vp, vp, vp, vp],
                              ctypes.c_int),
        "vmp_sphere_hits": ([vp, vp, c_i64, c_i64, ctypes.c_float, vp, vp], ctypes.c_int),
        "vmp_pair_clear": ([vp, vp, c_i64, c_i64, ctypes.c_float, vp, vp], ctypes.c_int),
        "vmp_knn": ([vp, c_i64, c_i64, c_i32, vp, c_i64, c_i64, vp, c_i32, vp, vp, vp],
                    ctypes.c_int),
        "vmp_nn_distances": ([vp, c_i64, c_i64, c_i32, vp, c_i64, c_i64, vp, c_i64, vp],
                             ctypes.c_int),
        "vmp_debug_motion_trace": ([vp, c_i64], c_i64),
        "vmp_set_device": ([c_i32], ctypes.c_int),
        "vmp_device_info": ([ctypes.POINTER(c_i32), ctypes.POINTER(c_i32)], ctypes.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _LIB = L
    return L


def check(rc: int) -> None:
    """Map a vmp status to the reference's exception types."""
    if rc == VMP_OK:
        return
    msg = lib().vmp_last_error().decode(errors="replace")
    if rc == VMP_EARG:
        raise ValueError(msg)
    raise RuntimeError(f"vmp error {rc}: {msg}")
