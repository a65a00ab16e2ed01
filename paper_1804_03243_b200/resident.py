"""Decoding from device-resident acoustic costs (C-ABI lb_decode_batch_device).

The acoustic model of an ASR pipeline leaves its log-likelihoods in HBM; this
entry point decodes straight from those buffers without
the host round trip.  Inputs are CUDA float64 tensors (torch is only the
allocator here); results are the 1-best fields plus the device timings.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .errors import DeviceError
from ._lib import P32, P64, PD, PV, ptr
from .decoder import DecodeConfig, _raise_status, device_graph, result_timing


def decode_batch_resident(wfst, tensors, config: DecodeConfig | None = None, stream=None,
                          want_lattice: bool = False):
    """Decode CUDA f64 (or f32) tensors [T_u, D]; returns (list of dicts, timing dict)."""
    cfg = config if config is not None else DecodeConfig()
    cfg.validate()
    n = len(tensors)
    if n == 0:
        return [], {}
    D = int(tensors[0].shape[1])
    dt = str(tensors[0].dtype)
    for t in tensors:
        if not t.is_cuda or str(t.dtype) != dt or dt not in ("torch.float64", "torch.float32") \
                or not t.is_contiguous() or t.dim() != 2 or int(t.shape[1]) != D:
            raise DeviceError("resident decode needs contiguous CUDA float64 or float32 [T, D] tensors "
                              "of one dtype")
    g = device_graph(wfst, cfg.device)
    L = _lib.lib()
    T = np.asarray([int(t.shape[0]) for t in tensors], dtype=np.int32)
    c = cfg.to_c(want_lattice, False)
    res = PV()
    sp = C.c_void_p(stream.cuda_stream) if stream is not None else None
    if dt == "torch.float32":
        # f32 log-likelihoods (an acoustic model's output), widened exactly on the
        # device: results equal decoding the f64-widened matrices
        PF = C.POINTER(C.c_float)
        fptrs = (PF * n)(*[C.cast(C.c_void_p(t.data_ptr()), PF) for t in tensors])
        rc = L.lb_decode_batch_device_f32(g.handle, n, fptrs, ptr(T, P32), D, C.byref(c), sp, C.byref(res))
    else:
        cptrs = (PD * n)(*[C.cast(C.c_void_p(t.data_ptr()), PD) for t in tensors])
        rc = L.lb_decode_batch_device(g.handle, n, cptrs, ptr(T, P32), D, C.byref(c), sp, C.byref(res))
    _raise_status(rc, _lib.last_error())
    try:
        out = []
        st, tc, part = C.c_int32(), C.c_double(), C.c_int32()
        plen, ntok, nlat = C.c_int64(), C.c_int64(), C.c_int64()
        cnt = np.zeros(8, dtype=np.int64)
        for u in range(n):
            L.lb_result_status(res, u, C.byref(st), None, 0, None, 0)
            L.lb_result_best(res, u, C.byref(tc), C.byref(part), C.byref(plen), C.byref(ntok),
                             C.byref(nlat))
            L.lb_result_counters(res, u, ptr(cnt, P64))
            path = np.zeros(plen.value, dtype=np.int32)
            L.lb_result_path(res, u, ptr(path, P32))
            out.append({"status": st.value, "total_cost": tc.value, "partial": bool(part.value),
                        "path": path, "counters": cnt.copy()})
        tm = result_timing(res)
        ph = np.zeros(8)
        L.lb_result_phases(res, ptr(ph, PD))
        names = ("emit", "winners", "max_active", "epsilon", "aggregate", "lattice", "turnover",
                 "frame0_final")
        tm["phases_ms"] = dict(zip(names, ph.tolist()))
        wb, wn = np.zeros(8), np.zeros(8)
        L.lb_result_warp_phases(res, ptr(wb, PD), ptr(wn, PD))
        tm["warp_busy_ms"] = dict(zip(names, wb.tolist()))
        tm["warp_samples"] = dict(zip(names, wn.tolist()))
        return out, tm
    finally:
        L.lb_result_free(res)
