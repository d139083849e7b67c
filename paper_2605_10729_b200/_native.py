"""ctypes binding of libpifb200.so (the C ABI declared in include/pif_b200.h).

There is no fallback: if the library is missing or fails to load, every
product entry point raises.  Build it with ``python -m paper_2605_10729_b200.build``
(or ``__graft_entry__.build()``); the .so lives in-tree next to this file.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PIF_B200_LIB", os.path.join(_HERE, "libpifb200.so"))

PIF_OK, PIF_ERR_VALUE, PIF_ERR_CUDA, PIF_ERR_STATE = 0, 1, 2, 3
PIF_PERMUTE_POSITIONS, PIF_PERMUTE_VELOCITIES, PIF_PERMUTE_RESET = 1, 2, 4
SHAPE = {"delta": 0, "cic": 1}
EXT = {"none": 0, "quadrupole": 1}

_lock = threading.Lock()
_lib = None


class NativeError(RuntimeError):
    """CUDA / cuFFT failure inside libpifb200."""


class pif_soa_t(ctypes.Structure):
    _fields_ = [("x", ctypes.c_void_p), ("y", ctypes.c_void_p), ("z", ctypes.c_void_p),
                ("vx", ctypes.c_void_p), ("vy", ctypes.c_void_p), ("vz", ctypes.c_void_p),
                ("id", ctypes.c_void_p), ("count", ctypes.c_int64)]


class pif_plan_desc_t(ctypes.Structure):
    _fields_ = [("N", ctypes.c_int), ("L", ctypes.c_double), ("eps", ctypes.c_double),
                ("w", ctypes.c_int), ("beta", ctypes.c_double), ("n_up", ctypes.c_int),
                ("deconv", ctypes.c_void_p), ("kvec", ctypes.c_void_p),
                ("shape_cic", ctypes.c_void_p), ("inv_L3", ctypes.c_double),
                ("half_L3", ctypes.c_double)]


_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_D = ctypes.c_double
_I = ctypes.c_int
_SOA = ctypes.POINTER(pif_soa_t)
_D3 = ctypes.POINTER(ctypes.c_double)

SIGNATURES = {
    "pif_last_error": ([], ctypes.c_char_p),
    "pif_abi_version": ([], _I),
    "pif_plan_create": ([ctypes.POINTER(pif_plan_desc_t), _I, ctypes.POINTER(_P)], _I),
    "pif_plan_destroy": ([_P], _I),
    "pif_plan_device_bytes": ([_P], _I64),
    "pif_es_poly_info": ([_I, _D, _D3, ctypes.POINTER(ctypes.c_int)], _I),
    "pif_wrap_points": ([_P, _P, _P, _P, _I64, _P], _I),
    "pif_bin_keys": ([_P, _SOA, _P, _P, _P], _I),
    "pif_bin_scatter": ([_P, _SOA, _SOA, _P, _P, _I, _P], _I),
    "pif_spread_sorted": ([_P, _SOA, _P, _D, _P], _I),
    "pif_bin_perm": ([_P, _P, _P, _I64, _P, _P], _I),
    "pif_spread_perm": ([_P, _SOA, _P, _P, _D, _P], _I),
    "pif_interp_push_perm": ([_P, _SOA, _P, _SOA, _D, _D, _D3, _D3, _I, _I, _P, _P, _P, _P], _I),
    "pif_interp_split": ([_P, _SOA, _P, _I64, _P], _I),
    "pif_push_ids": ([_P, _P, _P, _I64, _I64, _I64, _D, _D, _D3, _D3, _I, _I, _P, _P], _I),
    "pif_split_supported": ([_P], _I),
    "pif_set_spread_merge": ([_P, _I], _I),
    "pif_spread_merge_used": ([_P], _I),
    "pif_grid_to_modes": ([_P, _P, _P], _I),
    "pif_solve_fields": ([_P, _P, _I, _P, _P, _P], _I),
    "pif_fields_from_modes": ([_P, _P, _P, _P, _I, _P, _P], _I),
    "pif_field_energy": ([_P, _P, _P, _P], _I),
    "pif_poisson": ([_P, _P, _P, _P, _P, _P], _I),
    "pif_interp_push": ([_P, _SOA, _D, _D, _D3, _D3, _I, _I, _P, _P, _P, _P], _I),
    "pif_interp_sorted": ([_P, _SOA, _P, _P], _I),
    "pif_interp_perm": ([_P, _SOA, _P, _P, _P], _I),
    "pif_particle_diag": ([_P, _SOA, _I, _P, _P], _I),
    "pif_soa_to_aos": ([_P, _SOA, _I64, _P, _P, _P], _I),
    "pif_type1_complex": ([_P, _P, _P, _I64, _P, _P], _I),
    "pif_type2_complex": ([_P, _P, _P, _I64, _P, _P], _I),
    "pif_probe_fp64": ([_P, _I, _I, _I, _P, _D3], _I),
    "pif_debug_phase_cycles": ([_P], _I),
    "pif_load_aos": ([_P, _P, _P, _I64, _SOA, _P, _P, _P], _I),
    "pif_load_aos_velocities": ([_P, _P, _SOA, _P], _I),
    "pif_set_id_order_output": ([_P, _P, _P, _I64], _I),
    "pif_set_weight_cache": ([_P, _I], _I),
    "pif_type1_complex_sorted": ([_P, _SOA, _P, _P, _P, _P], _I),
    "pif_type2_complex_sorted": ([_P, _P, _SOA, _P, _P], _I),
    "pif_sample_landau_axis": ([_P, _P, _I64, _I64, _D, _D, _D, _P, _I64, _P, _P], _I),
    "pif_set_deterministic": ([_P, _I], _I),
    "pif_is_deterministic": ([_P], _I),
    "pif_push_aggregated": ([_P], _I),
    "pif_permute": ([_P, _SOA, _P, _SOA, _I, _P], _I),
    "pif_nccl_version": ([ctypes.POINTER(ctypes.c_int)], _I),
    "pif_comm_init_all": ([_I, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(_P)], _I),
    "pif_allreduce_f64": ([_P, _P, _I64, _P], _I),
    "pif_comm_destroy": ([_P], _I),
    "pif_fft_timing": ([_P, _I], _I),
    "pif_fft_times": ([_P, _D3, _D3, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)],
                      _I),
    "pif_sample_normal": ([_P, _P, _I64, _I64, _I64, _D, _D, _I, _D, _P, _I64, _P, _P], _I),
}


def load():
    """Load libpifb200.so and declare every exported function; raise if absent."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"{LIB_PATH} is missing: build the CUDA extension first "
                    "(python -m paper_2605_10729_b200.build); there is no CPU fallback")
            lib = ctypes.CDLL(LIB_PATH)
            # an A/B build named by PIF_B200_LIB may predate newer entry
            # points; the in-tree library must export all of them
            ab = "PIF_B200_LIB" in os.environ
            for name, (args, res) in SIGNATURES.items():
                if ab and not hasattr(lib, name):
                    continue
                fn = getattr(lib, name)
                fn.argtypes = args
                fn.restype = res
            _lib = lib
    return _lib


def check(rc: int, what: str = "") -> None:
    if rc == PIF_OK:
        return
    msg = load().pif_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc == PIF_ERR_VALUE:
        raise ValueError(text)
    raise NativeError(text)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)


def ptr(t) -> int:
    """Device pointer of a torch tensor (None -> NULL)."""
    return None if t is None else t.data_ptr()


def stream_handle(device=None) -> int:
    import torch
    return torch.cuda.current_stream(device).cuda_stream


def soa(x, y, z, vx=None, vy=None, vz=None, ids=None, count=None) -> pif_soa_t:
    n = int(count if count is not None else x.shape[0])
    return pif_soa_t(ptr(x), ptr(y), ptr(z), ptr(vx), ptr(vy), ptr(vz), ptr(ids), n)


def soa_from_store(buf, ids, count) -> pif_soa_t:
    """View of a (6, cap) float64 buffer + int64 ids as a pif_soa_t."""
    return pif_soa_t(ptr(buf[0]), ptr(buf[1]), ptr(buf[2]), ptr(buf[3]), ptr(buf[4]),
                     ptr(buf[5]), ptr(ids), int(count))


def d3(v) -> ctypes.Array:
    arr = (ctypes.c_double * 3)(*[float(a) for a in v])
    return arr


def loaded_path() -> str | None:
    return LIB_PATH if _lib is not None else None
