"""ctypes binding of libtbf_b200.so (C ABI: include/oiobf_b200.h).

The product path has no CPU fallback: if the library is missing or no sm_100
device is present, every compute call raises.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libtbf_b200.so")

i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")


class OiobfError(RuntimeError):
    pass


class KernelSpecC(C.Structure):
    _fields_ = [("kind", C.c_int32), ("d", C.c_int32), ("n", C.c_int64), ("bitrev", C.c_int32), ("seed", C.c_uint32),
                ("kappa", C.c_double), ("offset", C.c_double * 3)]


class ProxyStrategyC(C.Structure):
    _fields_ = [("mode", C.c_int32), ("pad_", C.c_int32), ("q", C.c_int64), ("max_retries", C.c_int64),
                ("row_cap", C.c_int64)]


# Every symbol include/oiobf_b200.h declares (tests/test_capi.py checks them).
EXPORTS = [
    "oiobf_last_error", "oiobf_set_device", "oiobf_device_info", "oiobf_column_id_batch",
    "oiobf_select_proxies_count", "oiobf_derive_seed", "oiobf_subtensor_at", "oiobf_mode_product_blockdiag",
    "oiobf_tbf_construct", "oiobf_tbf_destroy", "oiobf_tbf_contract", "oiobf_tbf_contract_device",
    "oiobf_tbf_memory", "oiobf_tbf_info", "oiobf_tbf_export", "oiobf_tbf_timings", "oiobf_tbf_plan_stats",
    "oiobf_tbf_profile_contract", "oiobf_dense_rows", "oiobf_tbf_check_finite",
    "oiobf_tbf_shard_begin", "oiobf_tbf_shard_set_owners", "oiobf_tbf_shard_level", "oiobf_tbf_umid_info", "oiobf_tbf_umid_export",
    "oiobf_tbf_umid_import", "oiobf_tbf_set_exchange", "oiobf_tbf_contract_phase",
    "oiobf_tbf_set_apply_engine", "oiobf_tbf_apply_engine", "oiobf_tbf_save", "oiobf_tbf_load",
    "oiobf_tbf_contract_async", "oiobf_tbf_set_peer_exchange", "oiobf_device_alloc", "oiobf_device_free",
    "oiobf_ipc_handle", "oiobf_ipc_open", "oiobf_ipc_close", "oiobf_memcpy", "oiobf_synchronize",
    "oiobf_tbf_copy_owned", "oiobf_tbf_set_core_format",
    "oiobf_tbf_export_cores",
    "oiobf_tbf_profile_core_cold", "oiobf_fp64_peak",
]

_lock = threading.Lock()
_lib = None


def load(path: str = LIB_PATH):
    """Load (once) and declare signatures.  Raises if the library is missing."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise OiobfError(f"{path} is missing: run __graft_entry__.build() (no CPU fallback exists)")
        L = C.CDLL(path)
        L.oiobf_last_error.restype = C.c_char_p
        L.oiobf_set_device.argtypes = [C.c_int]
        L.oiobf_device_info.argtypes = [i64p]
        L.oiobf_derive_seed.restype = C.c_uint64
        L.oiobf_derive_seed.argtypes = [C.c_uint64, u64p, C.c_int32]
        L.oiobf_select_proxies_count.argtypes = [C.c_int64, C.c_int64, C.c_int32, C.c_uint64, i64p, i64p]
        L.oiobf_column_id_batch.argtypes = [C.c_int64, i64p, i64p, i64p, f64p, C.c_double, C.c_void_p, i64p, i64p,
                                            i64p, i64p, f64p, i64p, i32p, f64p]
        L.oiobf_subtensor_at.argtypes = [C.POINTER(KernelSpecC), i64p, i64p, f64p]
        L.oiobf_mode_product_blockdiag.argtypes = [C.c_int32, i64p, f64p, C.c_int32, C.c_int32, i64p, i64p, f64p,
                                                   C.c_int32, f64p]
        L.oiobf_tbf_construct.argtypes = [C.POINTER(KernelSpecC), C.c_int32, C.c_double, C.POINTER(ProxyStrategyC),
                                          C.c_uint64, C.POINTER(C.c_void_p)]
        L.oiobf_tbf_destroy.argtypes = [C.c_void_p]
        L.oiobf_tbf_contract.argtypes = [C.c_void_p, f64p, f64p, C.c_int64]
        L.oiobf_tbf_contract_device.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]
        L.oiobf_tbf_contract_async.argtypes = [C.c_void_p, f64p, f64p, C.c_int64, C.c_void_p]
        L.oiobf_tbf_memory.argtypes = [C.c_void_p, i64p]
        L.oiobf_tbf_set_apply_engine.argtypes = [C.c_void_p, C.c_int32]
        L.oiobf_tbf_set_core_format.argtypes = [C.c_void_p, C.c_int32]
        L.oiobf_tbf_save.argtypes = [C.c_void_p, C.c_char_p]
        L.oiobf_tbf_load.argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]
        L.oiobf_tbf_apply_engine.argtypes = [C.c_void_p, C.POINTER(C.c_int32)]
        L.oiobf_tbf_info.argtypes = [C.c_void_p, i64p]
        L.oiobf_tbf_export.argtypes = [C.c_void_p] + [C.c_void_p] * 10
        L.oiobf_tbf_timings.argtypes = [C.c_void_p, f64p]
        L.oiobf_tbf_plan_stats.argtypes = [C.c_void_p, i64p]
        L.oiobf_tbf_profile_contract.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, f64p]
        L.oiobf_tbf_check_finite.argtypes = [C.c_void_p, i64p]
        L.oiobf_dense_rows.argtypes = [C.POINTER(KernelSpecC), f64p, C.c_int64, C.c_int64, i64p, f64p]
        L.oiobf_tbf_export_cores.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.oiobf_tbf_profile_core_cold.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p,
                                                  C.c_void_p, C.c_int64, f64p]
        L.oiobf_fp64_peak.argtypes = [f64p]
        _lib = L
        return L


def check(rc: int) -> None:
    if rc != 0:
        msg = _lib.oiobf_last_error().decode()
        if rc == 1:
            raise ValueError(msg)  # std::invalid_argument in the reference
        raise OiobfError(msg)


def spec_c(spec) -> KernelSpecC:
    off = list(spec.offset) + [0.0] * (3 - len(spec.offset))
    return KernelSpecC(spec.kind, spec.d, spec.n, int(spec.bitrev), int(getattr(spec, "seed", 0)) & 0xFFFFFFFF,
                       spec.kappa, (C.c_double * 3)(*off[:3]))


def ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)
