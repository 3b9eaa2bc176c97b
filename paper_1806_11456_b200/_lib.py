"""ctypes binding of the C-ABI (include/taudg.h) — the only way the product
reaches the GPU.  There is no CPU fallback: if the shared library is missing
or no CUDA device is present, every device call raises DeviceError.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import ConfigError, DeviceError, MeshError

_HERE = os.path.dirname(os.path.abspath(__file__))
RK_TRACES_FRESH = 1   # include/taudg.h TDG_RK_TRACES_FRESH
# TDG_LIB_PATH: development override (A/B builds of the same C-ABI)
LIB_PATH = os.environ.get("TDG_LIB_PATH") or os.path.join(_HERE, "_taudg.so")

_i32, _i64, _dbl = C.c_int32, C.c_int64, C.c_double
_pd, _pi32, _pi64 = C.POINTER(C.c_double), C.POINTER(C.c_int32), C.POINTER(C.c_int64)


class PlanDesc(C.Structure):
    _fields_ = [
        ("law", _i32), ("params", _dbl * 8), ("family", _i32),
        ("tables", _pd), ("tables_len", _i64),
        ("nslots", _i32), ("orders", _pi32), ("elem_id", _pi32), ("node_off", _pi64),
        ("metric_off", _pi64), ("affine", _pi32), ("metrics", _pd), ("metrics_len", _i64),
        ("sizes", _pd),
        ("side_off", _pi64), ("side_nodes", _i64), ("side_geo", _pd),
        ("nfaces", _i32), ("face_info", _pi32), ("face_geo_off", _pi64), ("face_geo", _pd),
        ("face_geo_len", _i64),
        ("side_info", _pi32), ("mtr_nodes", _i64),
        ("nbfaces", _i32), ("bface_info", _pi32), ("ghost_off", _pi64), ("ghost", _pd),
        ("ghost_len", _i64),
    ]


class TransferDesc(C.Structure):
    _fields_ = [
        ("nslots", _i32), ("nv", _i32), ("tables", _pd), ("tables_len", _i64),
        ("fine_orders", _pi32), ("fine_elem_id", _pi32), ("fine_node_off", _pi64),
        ("coarse_orders", _pi32), ("coarse_elem_id", _pi32), ("coarse_node_off", _pi64),
    ]


_VP = C.c_void_p
SIGNATURES = {
    "tdg_plan_create": ([C.POINTER(PlanDesc), C.POINTER(_VP)], C.c_int),
    "tdg_plan_destroy": ([_VP], C.c_int),
    "tdg_plan_size": ([_VP, _pi64, _pi32], C.c_int),
    "tdg_apply": ([_VP, _VP, _VP, C.c_int, _VP], C.c_int),
    "tdg_m_inv_apply": ([_VP, _VP, _VP, _VP, C.c_int, _VP], C.c_int),
    "tdg_residual": ([_VP, _VP, _VP, _VP, _VP, _VP], C.c_int),
    "tdg_residual_host": ([_VP, _i32, C.POINTER(_VP), _VP, C.POINTER(_VP), _pd, _VP], C.c_int),
    "tdg_tau": ([_VP, _VP, _VP, _VP, C.c_int, _VP], C.c_int),
    "tdg_element_dt": ([_VP, _VP, _dbl, _dbl, _VP, _VP, _VP], C.c_int),
    "tdg_rk3_stage": ([_VP, _VP, _VP, _VP, C.c_int, _VP, C.c_int, _VP, _VP, _VP], C.c_int),
    "tdg_rk3_stage_ex": ([_VP, _VP, _VP, _VP, C.c_int, _VP, C.c_int, _VP, _VP, C.c_int, _VP], C.c_int),
    "tdg_norm_inf": ([_VP, _VP, _VP, _VP, _VP], C.c_int),
    "tdg_check_finite": ([_VP, _VP, _VP, _VP], C.c_int),
    "tdg_transfer_create": ([C.POINTER(TransferDesc), C.POINTER(_VP)], C.c_int),
    "tdg_transfer_destroy": ([_VP], C.c_int),
    "tdg_restrict": ([_VP, _VP, _VP, _VP], C.c_int),
    "tdg_prolong": ([_VP, _VP, _VP, _VP], C.c_int),
    "tdg_prolong_add": ([_VP, _VP, _VP, _VP, _VP], C.c_int),
    "tdg_gradient": ([_VP, _VP, C.c_int, _VP, _VP], C.c_int),
    "tdg_loop_begin": ([_VP, _VP, C.POINTER(_VP)], C.c_int),
    "tdg_loop_test": ([_VP, _VP, _VP, _VP, _VP, _dbl, C.c_int, _VP, C.c_int], C.c_int),
    "tdg_loop_end": ([_VP], C.c_int),
    "tdg_stream_create": ([C.POINTER(_VP)], C.c_int),
    "tdg_volume_metrics": ([_i32, _pi32, _pd, _pi32, _pd, _pd, _pd, _pd, _pd], C.c_int),
    "tdg_stream_destroy": ([_VP], C.c_int),
    "tdg_plan_info": ([_VP, _pi32, _pi32, _pi32], C.c_int),
    "tdg_tau_from_avalue": ([_VP, _VP, _VP, _VP, _VP], C.c_int),
    "tdg_debug_copy": ([_VP, C.c_int, _VP, _pi64, _VP], C.c_int),
    "tdg_timing_enable": ([C.c_int], C.c_int),
    "tdg_timing_read": ([_pd, _pi64, C.c_int], C.c_int),
    "tdg_kernel_name": ([C.c_int], C.c_char_p),
    "tdg_last_error": ([], C.c_char_p),
    "tdg_version": ([], C.c_char_p),
}

_lib = None


def load():
    """Load the shared library (raises DeviceError if it is absent)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise DeviceError(
            f"CUDA extension {LIB_PATH} is missing; run `python -c 'import __graft_entry__ as g; g.build()'`"
        )
    lib = C.CDLL(LIB_PATH)
    for name, (args, res) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def check(rc: int, what: str = ""):
    if rc == 0:
        return
    msg = load().tdg_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc == 1:
        raise ConfigError(text)
    if rc == 2:
        raise MeshError(text)
    if rc == 5:
        raise ValueError(text)
    raise DeviceError(text)


def call(name: str, *args):
    check(getattr(load(), name)(*args), name)


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None -> NULL)."""
    if t is None:
        return None
    return t.data_ptr()


def stream_handle(device=None) -> int:
    import torch

    return torch.cuda.current_stream(device).cuda_stream


KERNEL_COUNT = 12


def timing_enable(on: bool = True):
    call("tdg_timing_enable", int(bool(on)))


def timing_read() -> dict:
    """{kernel name: (total ms, launches)} since the last read (clears)."""
    ms = (C.c_double * KERNEL_COUNT)()
    cnt = (C.c_int64 * KERNEL_COUNT)()
    call("tdg_timing_read", ms, cnt, KERNEL_COUNT)
    lib = load()
    return {lib.tdg_kernel_name(i).decode(): (ms[i], cnt[i]) for i in range(KERNEL_COUNT)}
