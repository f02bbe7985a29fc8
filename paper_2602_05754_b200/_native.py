"""ctypes loaders for the in-tree native libraries.

There is no Python or CPU fallback behind these handles: if a library is
missing or fails to load, every call raises NativeLibraryError.
"""
from __future__ import annotations

import ctypes
import os
import threading

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_DIR = os.path.join(_PKG, "lib")

_lock = threading.Lock()
_host = None
_device = None


class NativeLibraryError(RuntimeError):
    pass


class PfError(RuntimeError):
    """Raised for a nonzero PF_* status; `status` holds the code."""

    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status


PF_OK, PF_ERR_CONFIG, PF_ERR_DOMAIN, PF_ERR_NUMERICAL, PF_ERR_INVALID, PF_ERR_CUDA, PF_ERR_NCCL, PF_ERR_INTERNAL = range(8)


def _load(name: str) -> ctypes.CDLL:
    path = os.path.join(LIB_DIR, name)
    if not os.path.exists(path):
        raise NativeLibraryError(
            f"{path} is missing: run `python -m paper_2602_05754_b200.build` (there is no fallback path)")
    try:
        return ctypes.CDLL(path, mode=ctypes.RTLD_GLOBAL)
    except OSError as e:  # pragma: no cover - environment dependent
        raise NativeLibraryError(f"failed to load {path}: {e}") from e


c_int = ctypes.c_int
c_ll = ctypes.c_longlong
c_f = ctypes.c_float
c_d = ctypes.c_double
c_vp = ctypes.c_void_p
c_u64 = ctypes.c_uint64
c_cp = ctypes.c_char_p


def _sig(lib, name, argtypes, restype=c_int):
    fn = getattr(lib, name)
    fn.argtypes = argtypes
    fn.restype = restype
    return fn


def device() -> ctypes.CDLL:
    """libpf_device.so (needs torch imported first: ATen backs the attention glue)."""
    global _device
    with _lock:
        if _device is None:
            import torch  # noqa: F401  (loads libc10/libtorch_cuda the library links against)

            lib = _load("libpf_device.so")
            _sig(lib, "pf_gemm_bf16", [c_vp, c_int, c_ll, c_vp, c_int, c_ll, c_vp, c_ll, c_int, c_int, c_int,
                                       c_f, c_int, c_int, c_vp, c_int, c_vp])
            _sig(lib, "pf_gemm_dw_units", [c_vp, c_int, c_ll, c_vp, c_int, c_ll, c_vp, c_ll, c_int, c_int, c_int,
                                           c_f, c_vp, c_vp, c_int, c_vp, c_int, c_int, c_vp])
            _sig(lib, "pf_gemm_dw_pairs", [c_vp, c_ll, c_vp, c_ll, c_vp, c_ll, c_int, c_int, c_int, c_vp, c_vp,
                                           c_vp, c_int, c_int, c_vp])
            _sig(lib, "pf_gemm_dw_rowpairs", [c_vp, c_ll, c_vp, c_ll, c_vp, c_ll, c_int, c_int, c_int, c_vp, c_vp,
                                              c_vp, c_int, c_int, c_vp])
            _sig(lib, "pf_gemm_dw_dense", [c_vp, c_ll, c_vp, c_ll, c_vp, c_ll, c_int, c_int, c_int, c_vp, c_int,
                                           c_int, c_vp])
            _sig(lib, "pf_device_sm_count", [], c_int)
            _sig(lib, "pf_device_last_error", [], c_cp)
            from . import _device_sigs

            _device_sigs.register(lib, _sig)
            _device = lib
        return _device


def host() -> ctypes.CDLL:
    """libpf_host.so (pure C++ host layer; usable without a GPU)."""
    global _host
    with _lock:
        if _host is None:
            lib = _load("libpf_host.so")
            from . import _host_sigs

            _host_sigs.register(lib, _sig)
            _host = lib
        return _host


def check(rc: int, what: str = "") -> None:
    if rc != PF_OK:
        detail = ""
        try:
            if _host is not None:
                detail = _host.pf_last_error().decode()
        except Exception:  # pragma: no cover
            pass
        if rc == PF_ERR_CUDA and _device is not None:
            detail = _device.pf_device_last_error().decode() or detail
        raise PfError(rc, f"{what} failed with status {rc}: {detail}")
