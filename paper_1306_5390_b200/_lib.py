"""ctypes binding of ``libphgrms_cuda.so`` (the C ABI in include/phgrms_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (nvcc,
``-gencode arch=compute_100a,code=sm_100a``).  There is no CPU fallback: if
the library is missing, importing the compute API raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PHG_LIB_PATH") or os.path.join(HERE, "libphgrms_cuda.so")

PHG_OK, PHG_EINVAL, PHG_ECUDA, PHG_ENOMEM, PHG_ENODEV = 0, -1, -2, -3, -4

# every symbol include/phgrms_b200.h declares
EXPORTS = (
    "phg_abi_version", "phg_last_error", "phg_validate_params", "phg_device_count",
    "phg_set_device", "phg_launch_count", "phg_reset_launch_count", "phg_cardinality",
    "phg_denoise_pass", "phg_denoise", "phg_denoise_batch", "phg_synth_image",
    "phg_inject_sp_noise", "phg_max_fused_iterations", "phg_dev_fused_step",
    "phg_dev_denoise", "phg_dev_cardinality", "phg_dev_removal", "phg_finalize_stats",
    "phg_fused_kernel_name", "phg_residual_noise_count", "phg_sse", "phg_dev_residual_count", "phg_dev_sse",
    "phg_dev_synth_smooth", "phg_dev_inject_noise", "phg_denoise_sharded", "phg_dev_fused_step_mirrored",
    "phg_ipc_get_handle", "phg_ipc_open_handle", "phg_ipc_close", "phg_debug_rms", "phg_denoise_pgm_file",
    "phg_launch_plan",
)


class PhgParams(C.Structure):
    """phg_params == phgrms::DenoiseParams (denoise.hpp:34-52)."""
    _fields_ = [("alpha", C.c_int32), ("beta", C.c_int32), ("max_iterations", C.c_int32),
                ("card_threshold", C.c_int32), ("border", C.c_int32)]


class PhgPassStats(C.Structure):
    """phg_pass_stats == phgrms::PassStats (denoise.hpp:71-76)."""
    _fields_ = [("iteration", C.c_int32), ("_pad", C.c_int32), ("flagged", C.c_int64),
                ("replaced", C.c_int64), ("elapsed_ms", C.c_double)]


class PhgDevImage(C.Structure):
    _fields_ = [("data", C.c_void_p), ("pitch", C.c_int64), ("image_stride", C.c_int64),
                ("width", C.c_int32), ("rows", C.c_int32), ("n_images", C.c_int32),
                ("_pad", C.c_int32)]


class PhgHaloPeer(C.Structure):
    """phg_halo_peer: owned rows [lo, hi) mirrored to ptr + (row - row0) * pitch."""
    _fields_ = [("ptr", C.c_void_p), ("row0", C.c_int32), ("lo", C.c_int32), ("hi", C.c_int32),
                ("_pad", C.c_int32)]


class InvalidArgument(ValueError):
    """Raised where the reference throws std::invalid_argument (same text)."""


class CudaError(RuntimeError):
    pass


_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                " (there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name in EXPORTS:
            getattr(L, name)  # AttributeError if the ABI is incomplete
        L.phg_last_error.restype = C.c_char_p
        L.phg_launch_count.restype = C.c_int64
        L.phg_validate_params.argtypes = [C.POINTER(PhgParams)]
        L.phg_device_count.argtypes = [C.POINTER(C.c_int)]
        L.phg_cardinality.argtypes = [_u8p, C.c_int, C.c_int, C.c_int, C.c_int, _i32p]
        L.phg_denoise_pass.argtypes = [_u8p, C.c_int, C.c_int, _i32p, C.c_int, C.c_int,
                                       C.POINTER(PhgParams), _u8p, C.POINTER(PhgPassStats)]
        L.phg_denoise.argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(PhgParams), C.c_int,
                                  C.c_void_p, C.POINTER(PhgPassStats), C.POINTER(C.c_int)]
        L.phg_denoise_batch.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(PhgParams),
                                        C.c_void_p, C.POINTER(PhgPassStats), C.POINTER(C.c_int)]
        L.phg_denoise_sharded.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(PhgParams),
                                          C.POINTER(C.c_int), C.c_int, C.c_void_p, C.POINTER(PhgPassStats),
                                          C.POINTER(C.c_int)]
        L.phg_dev_fused_step_mirrored.argtypes = [C.POINTER(PhgDevImage), C.POINTER(PhgDevImage), C.c_int, C.c_int,
                                                  C.c_int, C.c_int, C.POINTER(PhgParams), C.c_int, C.c_int,
                                                  C.c_void_p, C.c_int, C.POINTER(PhgHaloPeer), C.c_int,
                                                  C.c_void_p]
        L.phg_ipc_get_handle.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(C.c_uint64)]
        L.phg_ipc_open_handle.argtypes = [C.c_void_p, C.c_uint64, C.POINTER(C.c_void_p)]
        L.phg_ipc_close.argtypes = [C.c_void_p, C.c_uint64]
        L.phg_synth_image.argtypes = [C.c_int, C.c_int, C.c_uint32, C.c_int, _u8p]
        L.phg_inject_sp_noise.argtypes = [_u8p, C.c_int, C.c_int, C.c_double, C.c_double, C.c_uint32,
                                          _u8p, C.c_void_p]
        L.phg_inject_sp_noise.restype = C.c_int64
        L.phg_dev_fused_step.argtypes = [C.POINTER(PhgDevImage), C.POINTER(PhgDevImage), C.c_int, C.c_int,
                                         C.c_int, C.c_int, C.POINTER(PhgParams), C.c_int, C.c_int,
                                         C.c_void_p, C.c_int, C.c_void_p]
        L.phg_dev_denoise.argtypes = [C.POINTER(PhgDevImage), C.POINTER(PhgDevImage), C.POINTER(PhgDevImage),
                                      C.POINTER(PhgParams), C.c_void_p, C.c_void_p]
        L.phg_dev_cardinality.argtypes = [C.POINTER(PhgDevImage), C.c_int, C.c_int, C.c_void_p, C.c_int64,
                                          C.c_void_p]
        L.phg_dev_removal.argtypes = [C.POINTER(PhgDevImage), C.c_void_p, C.c_int64, C.POINTER(PhgParams),
                                      C.POINTER(PhgDevImage), C.c_void_p, C.c_void_p]
        L.phg_finalize_stats.argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(PhgPassStats),
                                         C.POINTER(C.c_int)]
        L.phg_max_fused_iterations.argtypes = [C.c_int]
        L.phg_launch_plan.argtypes = [C.POINTER(PhgParams), C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int]
        L.phg_fused_kernel_name.argtypes = [C.POINTER(PhgParams), C.c_int]
        L.phg_fused_kernel_name.restype = C.c_char_p
        L.phg_residual_noise_count.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                               C.POINTER(C.c_uint64)]
        L.phg_debug_rms.argtypes = [C.c_int, C.c_uint32, C.c_void_p]
        L.phg_denoise_pgm_file.argtypes = [C.c_char_p, C.c_char_p, C.POINTER(PhgParams), C.c_void_p,
                                           C.POINTER(C.c_int)]
        L.phg_sse.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_uint64)]
        L.phg_dev_residual_count.argtypes = [C.POINTER(PhgDevImage), C.c_int, C.c_int, C.c_int, C.c_void_p,
                                             C.c_void_p]
        L.phg_dev_sse.argtypes = [C.POINTER(PhgDevImage), C.POINTER(PhgDevImage), C.c_void_p, C.c_void_p]
        L.phg_dev_synth_smooth.argtypes = [C.POINTER(PhgDevImage), C.c_int, C.c_int, C.c_uint64, C.c_void_p]
        L.phg_dev_inject_noise.argtypes = [C.POINTER(PhgDevImage), C.c_int, C.c_int, C.c_double, C.c_double,
                                           C.c_uint64, C.c_void_p, C.c_void_p]
        _LIB = L
    return _LIB


def check(rc: int) -> None:
    """Map a PHG_* return code to the reference's exception behaviour."""
    if rc == PHG_OK:
        return
    msg = lib().phg_last_error().decode()
    if rc == PHG_EINVAL:
        raise InvalidArgument(msg)
    if rc == PHG_ENOMEM:
        raise MemoryError(msg)
    raise CudaError(f"[{rc}] {msg}")
