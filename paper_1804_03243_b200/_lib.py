"""ctypes binding of liblatbeam_b200.so (include/latbeam_b200.h).

The native library is the product: there is no CPU fallback.  `lib()` raises
DeviceError when the shared object is missing or no CUDA device is visible, so a
misconfigured box fails loudly instead of silently computing on the host.
ctypes releases the GIL for the duration of every call.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import DeviceError

_HERE = os.path.dirname(os.path.abspath(__file__))
# LB_SO_PATH: load a variant build (tools/variants.sh experiments only)
SO_PATH = os.environ.get("LB_SO_PATH") or os.path.join(_HERE, "liblatbeam_b200.so")

P64, P32, PD, PU64, PV = (C.POINTER(C.c_int64), C.POINTER(C.c_int32), C.POINTER(C.c_double),
                          C.POINTER(C.c_uint64), C.c_void_p)

# Every symbol include/latbeam_b200.h declares, with (restype, argtypes).
SIGNATURES = {
    "lb_version": (C.c_int32, []),
    "lb_last_error": (C.c_char_p, []),
    "lb_device_count": (C.c_int32, []),
    "lb_graph_create": (C.c_int, [C.c_int32, C.c_int64, C.c_int64, C.c_int32, P64, P32, P32, P32,
                                  P32, PD, PD, C.POINTER(PV)]),
    "lb_graph_destroy": (C.c_int, [PV]),
    "lb_graph_device_bytes": (C.c_int64, [PV]),
    "lb_decode_batch": (C.c_int, [PV, C.c_int32, C.POINTER(PD), P32, C.c_int32, PV, C.POINTER(PV)]),
    "lb_decode_batch_device": (C.c_int, [PV, C.c_int32, C.POINTER(PD), P32, C.c_int32, PV, PV,
                                         C.POINTER(PV)]),
    "lb_decode_batch_device_f32": (C.c_int, [PV, C.c_int32, C.POINTER(C.POINTER(C.c_float)), P32, C.c_int32, PV,
                                             PV, C.POINTER(PV)]),
    "lb_decode_batch_multi": (C.c_int, [C.POINTER(PV), C.c_int32, C.c_int32, C.POINTER(PD), P32, C.c_int32,
                                        PV, C.POINTER(PV)]),
    "lb_shard_lpt": (C.c_int, [C.c_int32, P32, C.c_int32, P32]),
    "lb_result_bulk": (C.c_int, [PV, P32, PD, P32, P64, P64]),
    "lb_result_paths": (C.c_int, [PV, P32]),
    "lb_result_count": (C.c_int, [PV, P32]),
    "lb_result_status": (C.c_int, [PV, C.c_int32, P32, C.c_char_p, C.c_int32, C.c_char_p, C.c_int32]),
    "lb_result_best": (C.c_int, [PV, C.c_int32, PD, P32, P64, P64, P64]),
    "lb_result_path": (C.c_int, [PV, C.c_int32, P32]),
    "lb_result_tokens": (C.c_int, [PV, C.c_int32, P64, P32, PD, P32, P32, PU64]),
    "lb_result_lattice": (C.c_int, [PV, C.c_int32, P64, P32, P32, P32, PD]),
    "lb_result_counters": (C.c_int, [PV, C.c_int32, P64]),
    "lb_result_final_lattice": (C.c_int, [PV, C.c_int32, P64, P64, P64, P64]),
    "lb_result_final_arrays": (C.c_int, [PV, C.c_int32, PU64, P64, PD, P32, P32, P32, P32, PD, PD]),
    "lb_result_timing": (C.c_int, [PV, C.POINTER(C.c_float), C.POINTER(C.c_float),
                                   C.POINTER(C.c_float), C.POINTER(C.c_float), P32]),
    "lb_result_phases": (C.c_int, [PV, PD]),
    "lb_result_warp_phases": (C.c_int, [PV, PD, PD]),
    "lb_result_free": (None, [PV]),
    "lb_oracle_wer_batch": (C.c_int, [C.c_int32, C.c_int32, PV, P64]),
    "lb_result_final_arrays64": (C.c_int, [PV, C.c_int32, P64, P64, P64, PD, P64, P64, P64, P64, PD, PD]),
    "lb_lattice_text": (C.c_int64, [C.c_int64, C.c_int64, C.c_int64, P64, PD, C.c_int64, P64, P64, P64,
                                    P64, PD, PD, C.c_char_p, C.c_int64]),
    "lb_prune_lattice": (C.c_int, [C.c_int32, C.c_int32, P64, PD, P64, P32, P32, C.POINTER(C.c_uint8), PD, PD,
                                   PD, C.c_double, C.POINTER(C.c_uint8), PD, PD]),
    "lb_finalize_lattice": (C.c_int, [C.c_int32, C.c_int64, PU64, PU64, P32, P32, PD, PD, C.c_int64, C.c_int32,
                                      C.c_int32, C.c_int64, PD, C.POINTER(PV)]),
    "lb_expand_emitting": (C.c_int, [PV, P32, PD, C.c_int64, PD, C.c_int32, C.c_double, P32, PD,
                                     P64, PD]),
    "lb_expand_nonemitting": (C.c_int, [PV, P32, PD, C.c_int64, C.c_double, P32, PD, P64]),
}


class LbConfig(C.Structure):
    _fields_ = [("beam", C.c_double), ("lattice_beam", C.c_double), ("acoustic_scale", C.c_double),
                ("max_active", C.c_int64), ("max_tokens_per_frame", C.c_int64),
                ("max_lattice_arcs", C.c_int64), ("token_arena", C.c_int64),
                ("want_lattice", C.c_int32), ("collect_frame_packs", C.c_int32),
                ("lanes", C.c_int32), ("threads_per_lane", C.c_int32), ("ctas_per_lane", C.c_int32),
                ("keep_work_lattice", C.c_int32)]


_lib = None
_host_lib = None


def host_lib():
    """The library bound for host-only entry points (no device required)."""
    global _host_lib
    if _host_lib is None:
        _host_lib = load_symbols_only()
    return _host_lib


def load_symbols_only():
    """Open the library and bind every declared symbol (no device needed)."""
    if not os.path.exists(SO_PATH):
        raise DeviceError(f"native library {SO_PATH} is missing; run __graft_entry__.build()")
    L = C.CDLL(SO_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    return L


def lib():
    """The bound library; raises DeviceError if it cannot run here."""
    global _lib
    if _lib is None:
        L = load_symbols_only()
        if L.lb_device_count() < 1:
            raise DeviceError("no CUDA device visible: the B200 decoder has no CPU fallback")
        _lib = L
    return _lib


def last_error() -> str:
    return (lib().lb_last_error() or b"").decode()


def ptr(a, t):
    return a.ctypes.data_as(t)
