"""ctypes front-end of the CPU oracle (TEST INFRASTRUCTURE — never the product path).

Only tests/, `__graft_entry__.smoke()` and bench.py's CPU legs import this
module.  It loads `oracle/liblatbeam_oracle.so` (a serial C restatement of the
reference decoder, see latbeam_oracle.c for the file:line map) and returns
plain numpy results the parity tests compare against the CUDA path.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liblatbeam_oracle.so")

STATUS = {0: "OK", 1: "DECODE_FAILURE", 2: "USAGE", 3: "CAPACITY", 4: "INTERNAL"}


class _Graph(C.Structure):
    _fields_ = [("S", C.c_int64), ("A", C.c_int64), ("start", C.c_int32),
                ("off", C.POINTER(C.c_int64)), ("src", C.POINTER(C.c_int32)),
                ("dst", C.POINTER(C.c_int32)), ("il", C.POINTER(C.c_int32)),
                ("ol", C.POINTER(C.c_int32)), ("w", C.POINTER(C.c_double)),
                ("final_cost", C.POINTER(C.c_double))]


class _Config(C.Structure):
    _fields_ = [("beam", C.c_double), ("lattice_beam", C.c_double), ("acoustic_scale", C.c_double),
                ("max_active", C.c_int64), ("max_tokens_per_frame", C.c_int64),
                ("max_lattice_arcs", C.c_int64), ("want_lattice", C.c_int32),
                ("collect_frames", C.c_int32)]


_P64, _P32, _PD, _PU64, _PU8 = (C.POINTER(C.c_int64), C.POINTER(C.c_int32), C.POINTER(C.c_double),
                                C.POINTER(C.c_uint64), C.POINTER(C.c_uint8))


class _Result(C.Structure):
    _fields_ = [("status", C.c_int32), ("msg", C.c_char * 256), ("bound", C.c_char * 64),
                ("total_cost", C.c_double), ("partial", C.c_int32),
                ("n_words", C.c_int64), ("words", _P32),
                ("n_align", C.c_int64), ("align_il", _P32), ("align_fr", _P32),
                ("n_frames", C.c_int32), ("tok_off", _P64), ("tok_state", _P32),
                ("tok_cost", _PD), ("tok_pred_arc", _P64), ("tok_pred_idx", _P64),
                ("tok_pack", _PU64), ("cutoffs", _PD),
                ("lat_off", _P64), ("lat_arc", _P32), ("lat_from", _P32), ("lat_to", _P32),
                ("lat_ac", _PD), ("lat_extra", _PD), ("lat_pruned", _PU8), ("node_extra", _PD),
                ("fl_num_nodes", C.c_int64), ("fl_start", C.c_int64), ("fl_n_final", C.c_int64),
                ("fl_n_arcs", C.c_int64), ("fl_final_ids", _P64), ("fl_final_costs", _PD),
                ("fl_from", _P64), ("fl_to", _P64), ("fl_il", _P64), ("fl_ol", _P64),
                ("fl_g", _PD), ("fl_ac", _PD), ("fl_node_frame", _P64), ("fl_node_idx", _P64),
                ("n_tokens", C.c_int64), ("n_scan", C.c_int64), ("n_cand", C.c_int64),
                ("eps_front", C.c_int64), ("eps_scan", C.c_int64), ("eps_cand", C.c_int64),
                ("n_next", C.c_int64), ("n_lat", C.c_int64)]


_lib = None


def build() -> str:
    """Compile the oracle library in place (gcc; seconds)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO) or (os.path.getmtime(_SO) < os.path.getmtime(
                os.path.join(_HERE, "latbeam_oracle.c"))):
            build()
        L = C.CDLL(_SO)
        L.lbo_decode.argtypes = [C.POINTER(_Graph), _PD, C.c_int32, C.c_int32,
                                 C.POINTER(_Config), C.POINTER(_Result)]
        L.lbo_result_free.argtypes = [C.POINTER(_Result)]
        L.lbo_decode_batch_mt.argtypes = [C.POINTER(_Graph), C.c_int32, C.POINTER(_PD), _P32,
                                          C.c_int32, C.POINTER(_Config), C.c_int32, _PD, _P32, _P64]
        L.lbo_expand_emitting.argtypes = [C.POINTER(_Graph), _P32, _PD, C.c_int64, _PD, C.c_double,
                                          _P32, _PD, _PD]
        L.lbo_expand_emitting.restype = C.c_int64
        L.lbo_expand_nonemitting.argtypes = [C.POINTER(_Graph), _P32, _PD, C.c_int64, C.c_double,
                                             _P32, _PD]
        L.lbo_expand_nonemitting.restype = C.c_int64
        _lib = L
    return _lib


def _ptr(a, t):
    return a.ctypes.data_as(t)


class OracleGraph:
    """Keeps the contiguous CSR columns alive for the C structure."""

    def __init__(self, wfst):
        self.keep = [np.ascontiguousarray(wfst.arc_offsets, dtype=np.int64),
                     np.ascontiguousarray(wfst.arc_src, dtype=np.int32),
                     np.ascontiguousarray(wfst.arc_dst, dtype=np.int32),
                     np.ascontiguousarray(wfst.arc_ilabel, dtype=np.int32),
                     np.ascontiguousarray(wfst.arc_olabel, dtype=np.int32),
                     np.ascontiguousarray(wfst.arc_weight, dtype=np.float64),
                     np.ascontiguousarray(wfst.final_cost_array, dtype=np.float64)]
        off, src, dst, il, ol, w, fc = self.keep
        self.s = _Graph(int(wfst.num_states), len(src), int(wfst.start_state), _ptr(off, _P64),
                        _ptr(src, _P32), _ptr(dst, _P32), _ptr(il, _P32), _ptr(ol, _P32),
                        _ptr(w, _PD), _ptr(fc, _PD))


@dataclass
class OracleResult:
    status: int
    message: str
    bound: str
    words: list = field(default_factory=list)
    alignment: list = field(default_factory=list)
    total_cost: float = float("nan")
    partial: bool = False
    frames: list | None = None          # [(states, costs, pred_arc, pred_idx, packs)]
    cutoffs: np.ndarray | None = None
    blocks: list | None = None          # [(arc, from, to, ac, extra, pruned)] per block
    node_extra: list | None = None
    final: dict | None = None
    counters: dict = field(default_factory=dict)

    @property
    def ok(self) -> bool:
        return self.status == 0

    @property
    def frame_packs(self):
        return [(f[0], f[4]) for f in self.frames] if self.frames is not None else None


def _arr(p, n, dt):
    if n == 0:
        return np.empty(0, dtype=dt)
    return np.ctypeslib.as_array(p, shape=(n,)).astype(dt, copy=True)


def decode(wfst, costs, beam, lattice_beam=8.0, acoustic_scale=1.0, max_active=0,
           max_tokens_per_frame=1_000_000, max_lattice_arcs=1 << 40, want_lattice=True,
           collect_frames=True, graph: OracleGraph | None = None) -> OracleResult:
    L = lib()
    g = graph or OracleGraph(wfst)
    m = np.ascontiguousarray(getattr(costs, "costs", costs), dtype=np.float64)
    cfg = _Config(float(beam), float(lattice_beam), float(acoustic_scale), int(max_active),
                  int(max_tokens_per_frame), int(max_lattice_arcs), int(bool(want_lattice)),
                  int(bool(collect_frames)))
    r = _Result()
    L.lbo_decode(C.byref(g.s), _ptr(m, _PD), m.shape[0], m.shape[1], C.byref(cfg), C.byref(r))
    try:
        out = OracleResult(r.status, r.msg.decode(), r.bound.decode())
        out.counters = {k: getattr(r, k) for k in ("n_tokens", "n_scan", "n_cand", "eps_front",
                                                   "eps_scan", "eps_cand", "n_next", "n_lat")}
        if r.status != 0:
            return out
        out.words = _arr(r.words, r.n_words, np.int64).tolist()
        out.alignment = list(zip(_arr(r.align_il, r.n_align, np.int64).tolist(),
                                 _arr(r.align_fr, r.n_align, np.int64).tolist()))
        out.total_cost = r.total_cost
        out.partial = bool(r.partial)
        if r.n_frames:
            nf = r.n_frames
            toff = _arr(r.tok_off, nf + 1, np.int64)
            n = int(toff[-1])
            cols = [_arr(r.tok_state, n, np.int32), _arr(r.tok_cost, n, np.float64),
                    _arr(r.tok_pred_arc, n, np.int64), _arr(r.tok_pred_idx, n, np.int64),
                    _arr(r.tok_pack, n, np.uint64)]
            out.frames = [tuple(c[toff[f]:toff[f + 1]] for c in cols) for f in range(nf)]
            out.cutoffs = _arr(r.cutoffs, nf, np.float64)
            if want_lattice:
                loff = _arr(r.lat_off, nf + 1, np.int64)
                na = int(loff[-1])
                lc = [_arr(r.lat_arc, na, np.int64), _arr(r.lat_from, na, np.int64),
                      _arr(r.lat_to, na, np.int64), _arr(r.lat_ac, na, np.float64),
                      _arr(r.lat_extra, na, np.float64), _arr(r.lat_pruned, na, np.uint8).astype(bool)]
                out.blocks = [tuple(c[loff[b]:loff[b + 1]] for c in lc) for b in range(nf)]
                ne = _arr(r.node_extra, n, np.float64)
                out.node_extra = [ne[toff[f]:toff[f + 1]] for f in range(nf)]
                k, a = r.fl_n_final, r.fl_n_arcs
                nn = r.fl_num_nodes
                out.final = dict(num_nodes=nn, start=r.fl_start,
                                 final_ids=_arr(r.fl_final_ids, k, np.int64),
                                 final_costs=_arr(r.fl_final_costs, k, np.float64),
                                 from_=_arr(r.fl_from, a, np.int64), to=_arr(r.fl_to, a, np.int64),
                                 ilabel=_arr(r.fl_il, a, np.int64), olabel=_arr(r.fl_ol, a, np.int64),
                                 graph_cost=_arr(r.fl_g, a, np.float64),
                                 acoustic_cost=_arr(r.fl_ac, a, np.float64),
                                 node_frame=_arr(r.fl_node_frame, nn, np.int64),
                                 node_idx=_arr(r.fl_node_idx, nn, np.int64), num_frames=nf - 1)
        return out
    finally:
        L.lbo_result_free(C.byref(r))


def decode_batch_mt(wfst, matrices, beam, lattice_beam=8.0, acoustic_scale=1.0, max_active=0,
                    want_lattice=False, nthreads=None, graph: OracleGraph | None = None,
                    max_tokens_per_frame=1_000_000):
    """Many utterances over host threads; returns (total_costs, statuses, counters[n,8])."""
    L = lib()
    g = graph or OracleGraph(wfst)
    mats = [np.ascontiguousarray(getattr(m, "costs", m), dtype=np.float64) for m in matrices]
    n = len(mats)
    D = mats[0].shape[1]
    ptrs = (_PD * n)(*[_ptr(m, _PD) for m in mats])
    T = np.asarray([m.shape[0] for m in mats], dtype=np.int32)
    cfg = _Config(float(beam), float(lattice_beam), float(acoustic_scale), int(max_active),
                  int(max_tokens_per_frame), 1 << 40, int(bool(want_lattice)), 0)
    tc = np.zeros(n)
    st = np.zeros(n, dtype=np.int32)
    cnt = np.zeros((n, 8), dtype=np.int64)
    L.lbo_decode_batch_mt(C.byref(g.s), n, ptrs, _ptr(T, _P32), D, C.byref(cfg),
                          int(nthreads or os.cpu_count() or 1), _ptr(tc, _PD), _ptr(st, _P32),
                          _ptr(cnt, _P64))
    return tc, st, cnt


def expand_emitting(wfst, states, costs, acrow, beam):
    L = lib()
    g = OracleGraph(wfst)
    s = np.ascontiguousarray(states, dtype=np.int32)
    c = np.ascontiguousarray(costs, dtype=np.float64)
    row = np.ascontiguousarray(acrow, dtype=np.float64)
    os_ = np.empty(wfst.num_states, dtype=np.int32)
    oc = np.empty(wfst.num_states)
    cut = np.zeros(1)
    m = L.lbo_expand_emitting(C.byref(g.s), _ptr(s, _P32), _ptr(c, _PD), len(s), _ptr(row, _PD),
                              float(beam), _ptr(os_, _P32), _ptr(oc, _PD), _ptr(cut, _PD))
    return os_[:m].astype(np.int64), oc[:m].copy(), float(cut[0])


def expand_nonemitting(wfst, states, costs, cutoff):
    L = lib()
    g = OracleGraph(wfst)
    s = np.ascontiguousarray(states, dtype=np.int32)
    c = np.ascontiguousarray(costs, dtype=np.float64)
    os_ = np.empty(wfst.num_states, dtype=np.int32)
    oc = np.empty(wfst.num_states)
    m = L.lbo_expand_nonemitting(C.byref(g.s), _ptr(s, _P32), _ptr(c, _PD), len(s), float(cutoff),
                                 _ptr(os_, _P32), _ptr(oc, _PD))
    if m < 0:
        raise RuntimeError(f"oracle status {-m}")
    return os_[:m].astype(np.int64), oc[:m].copy()
