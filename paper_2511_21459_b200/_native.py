"""ctypes binding of the sm_100a library (include/tsdf_b200.h).

The product path is: Python host code -> this C ABI -> hand-written CUDA
kernels.  There is no CPU fallback: if the shared library is missing or no
CUDA device is visible, every operator raises.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

from .errors import (CapacityError, ConfigError, DatasetError, DeviceError, FormatError,
                     NotFoundError)

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "_lib" / "libtsdf_b200.so"
_lib = None

F64, F32, U8, U16 = 0, 1, 2, 3
MEM_HOST, MEM_DEVICE = 0, 1


class IntegrationStatsC(C.Structure):
    _fields_ = [("measurements", C.c_int64), ("skipped_invalid", C.c_int64),
                ("blocks_allocated", C.c_int64), ("blocks_touched", C.c_int64),
                ("voxels_updated", C.c_int64), ("observations", C.c_int64),
                ("no_valid_warning", C.c_int32), ("pad", C.c_int32)]


class MergeStatsC(C.Structure):
    _fields_ = [("candidates", C.c_int64), ("merged", C.c_int64)]


class MeshC(C.Structure):
    _fields_ = [("vertices", C.POINTER(C.c_double)), ("normals", C.POINTER(C.c_double)),
                ("colors", C.POINTER(C.c_double)), ("num_vertices", C.c_int64),
                ("triangles", C.POINTER(C.c_int64)), ("num_triangles", C.c_int64)]


def build(force: bool = False) -> Path:
    """Compile the CUDA sources for sm_100a (nvcc cross-compiles without a GPU)."""
    src = _PKG / "csrc"
    newest = max(p.stat().st_mtime for p in list(src.glob("*.cu")) + list(src.glob("*.cuh"))
                 + list(src.glob("*.h")) + [_PKG.parent / "include" / "tsdf_b200.h"])
    if force or not LIB_PATH.exists() or LIB_PATH.stat().st_mtime < newest:
        jobs = str(max(1, min(8, os.cpu_count() or 1)))
        subprocess.run(["make", "-s", "-j", jobs, "-C", str(src)], check=True)
    return LIB_PATH


def source_digest() -> str:
    """sha256 (16 hex) of the CUDA sources and the ABI header: identifies the
    build a profile was captured on (there is no .git on the GPU box)."""
    import hashlib
    h = hashlib.sha256()
    src = _PKG / "csrc"
    for p in sorted(list(src.glob("*.cu")) + list(src.glob("*.cuh")) + list(src.glob("*.h"))
                    + [src / "Makefile", _PKG.parent / "include" / "tsdf_b200.h"]):
        h.update(p.name.encode())
        h.update(p.read_bytes())
    return h.hexdigest()[:16]


_ptr = C.c_void_p
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


def lib():
    """The loaded native library; raises if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (this package has no CPU fallback)")
    L = C.CDLL(str(LIB_PATH))
    i32, i64, dbl = C.c_int32, C.c_int64, C.c_double
    L.tsdf_table_create.argtypes = [i64, i32, i32, dbl, i32, _i64p, _ptr, C.POINTER(_ptr)]
    L.tsdf_table_destroy.argtypes = [_ptr]
    L.tsdf_table_reset.argtypes = [_ptr]
    L.tsdf_table_set_shard.argtypes = [_ptr, i32, i32]
    L.tsdf_table_set_depth_scale.argtypes = [_ptr, C.c_double]
    L.tsdf_table_set_lidar_mode.argtypes = [_ptr, i32]
    L.tsdf_table_stream.argtypes = [_ptr, C.POINTER(_ptr)]
    L.tsdf_table_version.argtypes = [_ptr, C.POINTER(C.c_uint64)]
    L.tsdf_read_level_blocks.argtypes = [_ptr, i32, _ptr, i64, _ptr, _ptr, _ptr, _ptr]
    L.tsdf_depth_window_frames.argtypes = [_ptr, i32, _ptr, i32, _ptr, i32, i32, i32, i32, _f64p, _f64p,
                                           _f64p, dbl, dbl, i32, i32, _ptr]
    L.tsdf_depth_window_walk.argtypes = [_ptr, _ptr, _ptr, i64]
    L.tsdf_depth_window_update.argtypes = [_ptr, _ptr, i32, i64, dbl, dbl, dbl, i32, _ptr,
                                           C.POINTER(MergeStatsC)]
    L.tsdf_table_merge_audit.argtypes = [_ptr, C.POINTER(C.c_int64)]
    L.tsdf_integrate_depth.argtypes = [_ptr, _ptr, i32, _ptr, i32, i32, i32, i32, _f64p, _f64p,
                                       _f64p, dbl, dbl, C.POINTER(IntegrationStatsC)]
    L.tsdf_integrate_depth_batch.argtypes = [_ptr, i32, _ptr, i32, _ptr, i32, i32, i32, i32,
                                             _f64p, _f64p, _f64p, dbl, dbl,
                                             C.POINTER(IntegrationStatsC), C.POINTER(i32)]
    L.tsdf_integrate_depth_window.argtypes = [_ptr, i32, _ptr, i32, _ptr, i32, i32, i32, i32,
                                              _f64p, _f64p, _f64p, dbl, dbl,
                                              C.POINTER(IntegrationStatsC), C.POINTER(i32), dbl,
                                              dbl, dbl, i32, dbl, C.POINTER(MergeStatsC)]
    L.tsdf_integrate_depth_walk.argtypes = [_ptr, _ptr, i32, _ptr, i32, i32, i32, i32, _f64p,
                                            _f64p, _f64p, dbl, dbl, i32, i32, _ptr, i64, _i64p,
                                            C.POINTER(IntegrationStatsC)]
    L.tsdf_integrate_depth_keys.argtypes = [_ptr, _ptr, i64, C.POINTER(IntegrationStatsC)]
    L.tsdf_integrate_points.argtypes = [_ptr, _ptr, i32, _ptr, i32, i64, i32, _f64p, _f64p, dbl,
                                        dbl, C.POINTER(IntegrationStatsC)]
    L.tsdf_allocate_for_measurement.argtypes = [_ptr, _f64p, _f64p, dbl, _i64p, i64,
                                                C.POINTER(i64)]
    L.tsdf_apply_merges.argtypes = [_ptr, dbl, dbl, dbl, i32, C.POINTER(MergeStatsC)]
    L.tsdf_extract_mesh.argtypes = [_ptr, dbl, dbl, C.POINTER(MeshC)]
    L.tsdf_mesh_free.argtypes = [C.POINTER(MeshC)]
    L.tsdf_extract_mesh_begin.argtypes = [_ptr, dbl, dbl, C.POINTER(i64), C.POINTER(i64)]
    L.tsdf_extract_mesh_read.argtypes = [_ptr, _ptr, _ptr, _ptr, _ptr]
    L.tsdf_nn_distance.argtypes = [_ptr, i64, _ptr, i64, i32, _ptr, _ptr]
    L.tsdf_quadtree_build.argtypes = [_ptr, i32, i32, i32, dbl, i32, _ptr, _ptr, C.POINTER(i64), _ptr]
    L.tsdf_seed_splats.argtypes = [_ptr, i64, _ptr, i32, dbl, _ptr, i32, i32, i32, i32, _f64p, _f64p,
                                   _f64p, _ptr, _ptr, _ptr, _ptr, _ptr]
    L.tsdf_find_batch.argtypes = [_ptr, _i64p, i64, _i64p, np.ctypeslib.ndpointer(np.int32),
                                  np.ctypeslib.ndpointer(np.uint8)]
    L.tsdf_insert.argtypes = [_ptr, _i64p, i32, C.POINTER(i64)]
    L.tsdf_remove.argtypes = [_ptr, _i64p, C.POINTER(i32), _ptr, _ptr, _ptr, _ptr]
    L.tsdf_read_block.argtypes = [_ptr, _i64p, C.POINTER(i32), _ptr, _ptr, _ptr, _ptr]
    L.tsdf_write_block.argtypes = [_ptr, _i64p, _ptr, _ptr, _ptr, _ptr]
    L.tsdf_depth_keys.argtypes = [_ptr, _ptr, i32, i32, i32, i32, _f64p, _f64p, _f64p, dbl, _ptr,
                                  i64, C.POINTER(i64)]
    L.tsdf_scan_keys.argtypes = [_ptr, _ptr, i32, i64, i32, _f64p, _f64p, dbl, _ptr, i64,
                                 C.POINTER(i64)]
    L.tsdf_evict_level.argtypes = [_ptr, i32, _i64p, i64, _ptr, _ptr, _ptr, _ptr]
    L.tsdf_import_level.argtypes = [_ptr, i32, _i64p, i64, _ptr, _ptr, _ptr, _ptr]
    L.tsdf_live_count.argtypes = [_ptr, i32, C.POINTER(i64)]
    L.tsdf_export_level.argtypes = [_ptr, i32, i64, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr,
                                    C.POINTER(i64)]
    L.tsdf_last_error.restype = C.c_char_p
    L.tsdf_kernel_launches.restype = i64
    L.tsdf_kernel_launches.argtypes = [_ptr]
    L.tsdf_table_slots.restype = i64
    L.tsdf_table_slots.argtypes = [_ptr]
    L.tsdf_device_info.argtypes = [C.POINTER(i32)] * 3
    L.tsdf_table_probe_stats.argtypes = [_ptr, _i64p, C.POINTER(dbl)]
    L.tsdf_probe_length.argtypes = [_ptr, _i64p, C.c_int64, C.c_void_p]
    L.tsdf_table_compact.argtypes = [_ptr]
    L.tsdf_dda_blocks.argtypes = [_ptr, _ptr, i64, dbl, i32, C.POINTER(C.POINTER(i64)),
                                  C.POINTER(C.POINTER(i64)), C.POINTER(i64)]
    L.tsdf_merge_candidates.argtypes = [_ptr, dbl, dbl, dbl, C.POINTER(C.POINTER(i64)),
                                        C.POINTER(i64)]
    L.tsdf_collapse_vertices.argtypes = [_ptr, _ptr, _ptr, i64, _ptr, i64, dbl, C.POINTER(MeshC)]
    L.tsdf_mesh_block_summary.argtypes = [_ptr, _ptr, _ptr, _ptr, _ptr, _ptr, i64, C.POINTER(i64)]
    L.tsdf_mesh_emit_keys.argtypes = [_ptr, _ptr, _ptr, dbl, C.POINTER(MeshC)]
    L.tsdf_mesh_finish.argtypes = [_ptr, _ptr, _ptr, i64, _ptr, i64, dbl, dbl, C.POINTER(MeshC)]
    L.tsdf_free.argtypes = [_ptr]
    L.tsdf_profile_enable.argtypes = [_ptr, i32]
    L.tsdf_work_totals.argtypes = [_ptr, _i64p, i32]
    L.tsdf_profile_read.argtypes = [_ptr, i32, i32, C.c_char_p, i32, _f64p, _i64p, C.POINTER(i32)]
    _lib = L
    return L


_EXC = {2: ConfigError, 3: DatasetError, 4: CapacityError, 5: NotFoundError, 6: FormatError,
        8: ValueError, 9: DeviceError}


def check(status: int, what: str) -> None:
    if status:
        msg = lib().tsdf_last_error().decode(errors="replace")
        raise _EXC.get(status, DeviceError)(f"{what}: {msg}")


def device_info():
    a, b, c = C.c_int32(), C.c_int32(), C.c_int32()
    check(lib().tsdf_device_info(C.byref(a), C.byref(b), C.byref(c)), "device_info")
    return a.value, b.value, c.value


_CODES = {np.dtype(np.float64): F64, np.dtype(np.float32): F32, np.dtype(np.uint8): U8,
          np.dtype(np.uint16): U16}
_TORCH_CODES = {"torch.float64": F64, "torch.float32": F32, "torch.uint8": U8, "torch.uint16": U16}


def as_buffer(arr, allowed):
    """(pointer, dtype code, mem kind, keepalive) for a numpy array or a CUDA
    array (anything exposing __cuda_array_interface__, e.g. a torch tensor)."""
    codes = _CODES
    if type(arr) is np.ndarray:
        # fast path for the common case: a contiguous host array of a kernel dtype
        code = codes.get(arr.dtype)
        if code is not None and code in allowed and arr.flags.c_contiguous:
            return arr.__array_interface__["data"][0], code, MEM_HOST, arr
    elif type(arr).__module__ == "torch" and arr.is_cuda:
        # fast path: a torch tensor's __cuda_array_interface__ is rebuilt on
        # every access, which costs more than a frame's enqueue
        code = _TORCH_CODES.get(str(arr.dtype))
        if code is None or code not in allowed:
            raise ValueError(f"unsupported device dtype {arr.dtype}")
        if not arr.is_contiguous():
            raise ValueError("device arrays must be C-contiguous")
        return arr.data_ptr(), code, MEM_DEVICE, arr
    cai = getattr(arr, "__cuda_array_interface__", None)
    if cai is not None:
        dt = np.dtype(cai["typestr"])
        if dt not in codes or codes[dt] not in allowed:
            raise ValueError(f"unsupported device dtype {dt}")
        if cai.get("strides") is not None:
            exp = np.cumprod((1,) + tuple(cai["shape"][::-1]))[:-1][::-1] * dt.itemsize
            if tuple(cai["strides"]) != tuple(int(x) for x in exp):
                raise ValueError("device arrays must be C-contiguous")
        return cai["data"][0], codes[dt], MEM_DEVICE, arr
    a = np.asarray(arr)
    if a.dtype not in codes or codes[a.dtype] not in allowed:
        a = a.astype(np.float64)
    a = np.ascontiguousarray(a)
    return a.ctypes.data, codes[a.dtype], MEM_HOST, a
