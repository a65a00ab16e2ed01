"""Decoder API — drop-in for the reference's decode path, executed on the B200.

Mirrors `latbeam.decoder` (decoder.py:52-672): `DecodeConfig`, `DecodeResult`,
`decode_utterance`, `decode_batch`, `expand_emitting`, `expand_nonemitting`,
`compute_cutoff`, same argument meanings and the same exception classes.  All
decoding runs in liblatbeam_b200.so (csrc/); this module validates arguments,
uploads/caches the graph, calls the C-ABI, and reshapes results (state-sorted
token lists, words/alignment from the device's best path, lattice
canonicalisation).  There is no CPU fallback: without the native library or a
CUDA device every entry point raises DeviceError.
"""

from __future__ import annotations

import ctypes as C
import gc
import math
import threading
import time
import weakref
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import P32, P64, PD, PU64, PV, LbConfig, ptr
from .acoustics import CostMatrix
from .errors import (CapacityError, DecodeFailure, DeviceError, InternalInvariantError,
                     UsageError)
from .lattice import (STATUS_LIVE, STATUS_PRUNED, FinalLattice, FrameTokens, LazyWorkLattice,
                      WorkLattice, finalize_lattice)

_SCHEDULERS = ("static", "dynamic")


@dataclass
class DecodeConfig:
    """Knobs for one decode (decoder.py:52-89 of `latbeam`) plus device knobs.

    `num_workers`, `group_size`, `num_shards`, `prune_interval` and `scheduler`
    are validated for compatibility but only shape the reference's CPU threads;
    on the device every utterance is one lane (a CTA) and the lattice is pruned
    once from the final terminus (equal result, SURVEY.md §0 finding 3).

    Added: `max_active` (0 = off, the reference behaviour; histogram cutoff,
    DESIGN.md §3), `token_arena` (tokens kept per utterance over all frames,
    0 = auto), `lanes` (utterances in flight per launch, 0 = auto),
    `threads_per_lane` (CTA size 512/640/768, 0 = 640), `ctas_per_lane` (thread-block
    cluster size of a lane, 0 = auto), `device` (CUDA ordinal), `devices`
    (several ordinals: `decode_batch` shards the utterances over one graph replica
    per entry, longest first, and returns them in input order),
    `keep_work_lattice` (ship `DecodeResult.work_lattice`, every live arc with
    its extra cost, with the result; otherwise a lattice decode returns a
    `LazyWorkLattice` that re-decodes on first use -- same lattice, bit-exact).
    """

    beam: float = 14.0
    lattice_beam: float = 8.0
    acoustic_scale: float = 1.0
    num_workers: int = 1
    group_size: int = 32
    num_shards: int = 32
    prune_interval: int = 25
    max_tokens_per_frame: int = 1_000_000
    max_lattice_arcs: int = 1_000_000
    scheduler: str = "dynamic"
    max_active: int = 0
    token_arena: int = 0
    lanes: int = 0
    threads_per_lane: int = 0
    ctas_per_lane: int = 0
    device: int = 0
    keep_work_lattice: bool = False
    devices: tuple = ()

    def validate(self) -> None:
        if not (math.isfinite(self.beam) and self.beam > 0):
            raise UsageError("beam must be a positive finite number")
        if not (math.isfinite(self.lattice_beam) and self.lattice_beam >= 0):
            raise UsageError("lattice_beam must be >= 0")
        if not (math.isfinite(self.acoustic_scale) and self.acoustic_scale > 0):
            raise UsageError("acoustic_scale must be > 0")
        for name in ("num_workers", "group_size", "num_shards", "prune_interval",
                     "max_tokens_per_frame", "max_lattice_arcs"):
            if int(getattr(self, name)) < 1:
                raise UsageError(f"{name} must be >= 1")
        if self.scheduler not in _SCHEDULERS:
            raise UsageError(f"unknown scheduler {self.scheduler!r}; choose one of "
                             f"{', '.join(_SCHEDULERS)}")
        for name in ("max_active", "token_arena", "lanes", "threads_per_lane", "ctas_per_lane",
                     "device"):
            if int(getattr(self, name)) < 0:
                raise UsageError(f"{name} must be >= 0")
        devs = tuple(self.devices or ())
        if any(int(d) < 0 for d in devs):
            raise UsageError("devices must be CUDA ordinals >= 0")
        if int(self.threads_per_lane) not in (0, 512, 640, 768):
            raise UsageError("threads_per_lane must be 512, 640 or 768")
        if not 0 <= int(self.ctas_per_lane) <= 16:
            raise UsageError("ctas_per_lane must be in [0, 16]")

    def to_c(self, want_lattice: bool, collect_frame_packs: bool) -> LbConfig:
        return LbConfig(float(self.beam), float(self.lattice_beam), float(self.acoustic_scale),
                        int(self.max_active), int(self.max_tokens_per_frame),
                        int(self.max_lattice_arcs), int(self.token_arena), int(bool(want_lattice)),
                        int(bool(collect_frame_packs)), int(self.lanes), int(self.threads_per_lane),
                        int(self.ctas_per_lane), int(bool(self.keep_work_lattice)))


@dataclass
class DecodeResult:
    """What one utterance decodes to (decoder.py:92-103)."""

    words: list
    alignment: list
    total_cost: float
    partial: bool
    lattice: FinalLattice | None
    work_lattice: WorkLattice | None = None
    frame_packs: list | None = None
    timings: dict | None = None
    counters: dict | None = None


def compute_cutoff(best_cost: float, beam: float) -> float:
    """best + beam (decoder.py:182-186)."""
    if not (math.isfinite(beam) and beam > 0):
        raise UsageError("beam must be a positive finite number")
    return float(best_cost) + float(beam)


# ---------------------------------------------------------------------------
# Device graph replica
# ---------------------------------------------------------------------------

class DeviceGraph:
    """One graph's HBM replica (include/latbeam_b200.h lb_graph_create)."""

    def __init__(self, wfst, device: int = 0):
        L = _lib.lib()
        self.device = int(device)
        self.num_states = int(wfst.num_states)
        self.max_ilabel = int(wfst.max_ilabel)
        cols = [np.ascontiguousarray(wfst.arc_offsets, dtype=np.int64),
                np.ascontiguousarray(wfst.arc_src, dtype=np.int32),
                np.ascontiguousarray(wfst.arc_dst, dtype=np.int32),
                np.ascontiguousarray(wfst.arc_ilabel, dtype=np.int32),
                np.ascontiguousarray(wfst.arc_olabel, dtype=np.int32),
                np.ascontiguousarray(wfst.arc_weight, dtype=np.float64),
                np.ascontiguousarray(wfst.final_cost_array, dtype=np.float64)]
        h = PV()
        rc = L.lb_graph_create(self.device, self.num_states, len(cols[1]), int(wfst.start_state),
                               ptr(cols[0], P64), ptr(cols[1], P32), ptr(cols[2], P32),
                               ptr(cols[3], P32), ptr(cols[4], P32), ptr(cols[5], PD),
                               ptr(cols[6], PD), C.byref(h))
        _raise_status(rc, _lib.last_error())
        self.handle = h
        self._fin = weakref.finalize(self, L.lb_graph_destroy, h)

    @property
    def device_bytes(self) -> int:
        return int(_lib.lib().lb_graph_device_bytes(self.handle))


_graph_cache: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()
_cache_lock = threading.Lock()


def device_graph(wfst, device: int = 0, replica: int = 0) -> DeviceGraph:
    """The cached replica of `wfst` on `device` (uploaded once per graph object);
    `replica` > 0 asks for an additional, independent replica on the same device
    (own workspace and stream, so decodes on it run concurrently)."""
    if isinstance(wfst, DeviceGraph):
        return wfst
    with _cache_lock:
        per = _graph_cache.setdefault(wfst, {})
        key = (int(device), int(replica))
        g = per.get(key)
        if g is None:
            g = per[key] = DeviceGraph(wfst, device)
        return g


def device_replicas(wfst, devices) -> list:
    """One replica per entry of `devices` (a device listed twice gets two)."""
    seen: dict = {}
    out = []
    for d in devices:
        k = seen.get(int(d), 0)
        seen[int(d)] = k + 1
        out.append(device_graph(wfst, int(d), k))
    return out


def split_batch(lengths, n_shards: int) -> list:
    """Input indices of each shard under shard_lpt, ascending within a shard."""
    sh = shard_lpt(lengths, n_shards)
    return [np.flatnonzero(sh == k).tolist() for k in range(int(n_shards))]


def merge_in_order(n: int, shards: list, shard_results: list) -> list:
    """Inverse of split_batch: per-shard result lists back into input order."""
    out = [None] * int(n)
    for idx, res in zip(shards, shard_results):
        if len(idx) != len(res):
            raise UsageError("shard result count does not match its utterances")
        for i, r in zip(idx, res):
            out[i] = r
    if any(r is None for r in out) and n:
        raise UsageError("shards do not cover the batch")
    return out


def shard_lpt(lengths, n_shards: int) -> np.ndarray:
    """The longest-first utterance split the multi-device decode uses
    (lb_shard_lpt): shard index per utterance."""
    T = np.ascontiguousarray(lengths, dtype=np.int32)
    out = np.zeros(len(T), dtype=np.int32)
    rc = _lib.host_lib().lb_shard_lpt(len(T), ptr(T, P32), int(n_shards), ptr(out, P32))
    if rc != 0:
        raise UsageError("bad shard arguments")
    return out


def _raise_status(rc: int, msg: str, bound: str = "") -> None:
    if rc == 0:
        return
    if rc == 1:
        raise DecodeFailure(msg)
    if rc == 2:
        raise UsageError(msg)
    if rc == 3:
        raise CapacityError(bound or "--device-memory", msg)
    if rc == 4:
        raise InternalInvariantError(msg)
    raise DeviceError(msg)


# ---------------------------------------------------------------------------
# Full decode
# ---------------------------------------------------------------------------

def _matrix_array(m) -> np.ndarray:
    a = m.costs if hasattr(m, "costs") else np.asarray(m)
    a = np.ascontiguousarray(a, dtype=np.float64)
    if a.ndim != 2 or a.shape[0] < 1 or a.shape[1] < 1:
        raise UsageError("cost matrix must be 2-D with T >= 1 and D >= 1")
    return a


def decode_batch(wfst, matrices, config: DecodeConfig | None = None, want_lattice: bool = True,
                 collect_frame_packs: bool = False, collect_timings: bool = False,
                 errors: str = "raise") -> list:
    """Decode utterances as concurrent device lanes; results in input order.

    Mirrors decoder.py:644-672.  With errors="raise" (the reference behaviour)
    the first failing utterance's exception propagates; with errors="return"
    its slot holds the exception instead.
    """
    cfg = config if config is not None else DecodeConfig()
    cfg.validate()
    mats = [_matrix_array(m) for m in matrices]
    if not mats:
        return []
    D = mats[0].shape[1]
    if any(m.shape[1] != D for m in mats):
        raise UsageError("all cost matrices of a batch must have the same label count")
    if int(wfst.max_ilabel) > D:
        raise UsageError(f"graph uses input label {wfst.max_ilabel} but the cost matrix "
                         f"has only {D} columns")
    t0 = time.perf_counter()
    L = _lib.lib()
    n = len(mats)
    cptrs = (PD * n)(*[ptr(m, PD) for m in mats])
    T = np.asarray([m.shape[0] for m in mats], dtype=np.int32)
    c = cfg.to_c(want_lattice, collect_frame_packs)
    res = PV()
    devs = tuple(cfg.devices or ())
    if len(devs) > 1:
        # one replica per device, LPT shards on one host thread each (ctypes
        # releases the GIL; the threads live in the native library)
        reps = device_replicas(wfst, devs)
        hs = (PV * len(reps))(*[r.handle for r in reps])
        rc = L.lb_decode_batch_multi(hs, len(reps), n, cptrs, ptr(T, P32), D, C.byref(c), C.byref(res))
    else:
        g = device_graph(wfst, devs[0] if devs else cfg.device)
        rc = L.lb_decode_batch(g.handle, n, cptrs, ptr(T, P32), D, C.byref(c), C.byref(res))
    _raise_status(rc, _lib.last_error())
    try:
        out = collect_results(wfst, res, mats, cfg, want_lattice, collect_frame_packs,
                              collect_timings, t0)
    finally:
        L.lb_result_free(res)
    if errors == "raise":
        for r in out:
            if isinstance(r, Exception):
                raise r
    return out


def decode_utterance(wfst, matrix, config: DecodeConfig | None = None, want_lattice: bool = True,
                     collect_frame_packs: bool = False, collect_timings: bool = False) -> DecodeResult:
    """Decode one utterance (decoder.py:463-611)."""
    return decode_batch(wfst, [matrix], config, want_lattice, collect_frame_packs,
                        collect_timings)[0]


def result_timing(res) -> dict:
    f = [C.c_float() for _ in range(4)]
    nl = C.c_int32()
    _lib.lib().lb_result_timing(res, *[C.byref(x) for x in f], C.byref(nl))
    return {"decode_ms": f[0].value, "prune_ms": f[1].value, "h2d_ms": f[2].value,
            "d2h_ms": f[3].value, "launches": nl.value}


_COUNTER_NAMES = ("n_tokens", "n_scan", "n_cand", "eps_front", "eps_scan", "eps_cand", "n_next", "n_lat")


def collect_results(wfst, res, mats, cfg, want_lattice, collect_frame_packs, collect_timings, t0):
    """DecodeResults in input order.  The scalar results and every best path come
    back in two bulk calls (lb_result_bulk / lb_result_paths); words and
    alignments are sliced from one vectorised label lookup.  The cyclic garbage
    collector is paused while the results are built: a 4096-utterance batch
    allocates ~1.2M alignment tuples, and the collector's passes over them cost
    twice the construction itself."""
    was = gc.isenabled()
    gc.disable()
    try:
        return _collect_results(wfst, res, mats, cfg, want_lattice, collect_frame_packs, collect_timings, t0)
    finally:
        if was:
            gc.enable()


def _collect_results(wfst, res, mats, cfg, want_lattice, collect_frame_packs, collect_timings, t0):
    L = _lib.lib()
    tm = result_timing(res)
    n = len(mats)
    status = np.zeros(n, dtype=np.int32)
    total = np.zeros(n)
    part = np.zeros(n, dtype=np.int32)
    poff = np.zeros(n + 1, dtype=np.int64)
    cnt = np.zeros((n, 8), dtype=np.int64)
    _raise_status(L.lb_result_bulk(res, ptr(status, P32), ptr(total, PD), ptr(part, P32), ptr(poff, P64),
                                   ptr(cnt, P64)), _lib.last_error())
    paths = np.zeros(max(int(poff[-1]), 1), dtype=np.int32)
    _raise_status(L.lb_result_paths(res, ptr(paths, P32)), _lib.last_error())
    il_all = wfst.arc_ilabel[paths[:poff[-1]]]
    ol_all = wfst.arc_olabel[paths[:poff[-1]]]
    # words / emitting ilabels of every utterance from one mask each, split at the
    # utterances' boundaries in the compacted arrays
    wmask, imask = ol_all > 0, il_all > 0
    wcut = np.concatenate(([0], np.cumsum(wmask)))[poff]
    icut = np.concatenate(([0], np.cumsum(imask)))[poff]
    words_all = ol_all[wmask].tolist()
    ils_all = il_all[imask].tolist()
    wcut_l, icut_l = wcut.tolist(), icut.tolist()
    cnt_l = cnt.tolist()
    total_l, part_l, status_l = total.tolist(), part.tolist(), status.tolist()
    out = []
    msg = C.create_string_buffer(256)
    bound = C.create_string_buffer(64)
    st = C.c_int32()
    plen, ntok, nlat = C.c_int64(), C.c_int64(), C.c_int64()
    tcd, prt = C.c_double(), C.c_int32()
    for u, m in enumerate(mats):
        counters = dict(zip(_COUNTER_NAMES, cnt_l[u]))
        if status_l[u] != 0:
            L.lb_result_status(res, u, C.byref(st), msg, 256, bound, 64)
            try:
                _raise_status(st.value, msg.value.decode(), bound.value.decode())
            except Exception as exc:   # noqa: BLE001 - boxed per utterance
                out.append(exc)
            continue
        ils = ils_all[icut_l[u]:icut_l[u + 1]]
        r = DecodeResult(words_all[wcut_l[u]:wcut_l[u + 1]], list(zip(ils, range(len(ils)))), total_l[u],
                         bool(part_l[u]), None, None, None, None, counters)
        if want_lattice:
            r.lattice = _final_lattice(res, u, m.shape[0])
            if not cfg.keep_work_lattice:
                r.work_lattice = LazyWorkLattice(_work_thunk(wfst, m, cfg))
        if collect_frame_packs or (want_lattice and cfg.keep_work_lattice):
            L.lb_result_best(res, u, C.byref(tcd), C.byref(prt), C.byref(plen), C.byref(ntok), C.byref(nlat))
            try:
                _attach_lattice(r, wfst, res, u, m, cfg, ntok.value, nlat.value,
                                want_lattice and cfg.keep_work_lattice, collect_frame_packs)
            except Exception as exc:   # noqa: BLE001 - finalize failures are per utterance
                out.append(exc)
                continue
        if collect_timings:
            r.timings = {"token_passing": tm["decode_ms"] / 1e3,
                         "lattice_pruning": tm["prune_ms"] / 1e3,
                         "h2d": tm["h2d_ms"] / 1e3, "d2h": tm["d2h_ms"] / 1e3,
                         "launches": tm["launches"], "total": time.perf_counter() - t0}
        out.append(r)
    return out


def _work_thunk(wfst, m, cfg):
    """Re-decode one utterance keeping its work lattice (LazyWorkLattice)."""
    from dataclasses import replace

    def build():
        c = replace(cfg, keep_work_lattice=True, devices=(), lanes=0,
                    device=int(cfg.devices[0]) if cfg.devices else cfg.device)
        return decode_utterance(wfst, m, c, want_lattice=True).work_lattice
    return build


def _final_lattice(res, u, num_frames) -> FinalLattice:
    """The device-finalised lattice (lb_result_final_arrays) as a FinalLattice."""
    L = _lib.lib()
    nn, st, nf, na = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
    _raise_status(L.lb_result_final_lattice(res, u, C.byref(nn), C.byref(st), C.byref(nf), C.byref(na)),
                  _lib.last_error())
    nfr, nix = np.empty(nn.value, dtype=np.int64), np.empty(nn.value, dtype=np.int64)
    fids, fcs = np.empty(nf.value, dtype=np.int64), np.empty(nf.value)
    fr, to, il, ol = (np.empty(na.value, dtype=np.int64) for _ in range(4))
    gc, ac = np.empty(na.value), np.empty(na.value)
    _raise_status(L.lb_result_final_arrays64(res, u, ptr(nfr, P64), ptr(nix, P64), ptr(fids, P64), ptr(fcs, PD),
                                             ptr(fr, P64), ptr(to, P64), ptr(il, P64), ptr(ol, P64),
                                             ptr(gc, PD), ptr(ac, PD)), _lib.last_error())
    return FinalLattice(int(nn.value), int(st.value), fids, fcs, fr, to, il, ol, gc, ac, nfr, nix, num_frames)


def _attach_lattice(r, wfst, res, u, m, cfg, ntok, nlat, want_lattice, collect_frame_packs):
    L = _lib.lib()
    T = m.shape[0]
    F = T + 1
    foff = np.zeros(F + 1, dtype=np.int64)
    states = np.zeros(ntok, dtype=np.int32)
    costs = np.zeros(ntok)
    parc = np.zeros(ntok, dtype=np.int32)
    pidx = np.zeros(ntok, dtype=np.int32)
    packs = np.zeros(ntok, dtype=np.uint64)
    _raise_status(L.lb_result_tokens(res, u, ptr(foff, P64), ptr(states, P32), ptr(costs, PD),
                                     ptr(parc, P32), ptr(pidx, P32), ptr(packs, PU64)),
                  _lib.last_error())
    counts = np.diff(foff)
    fr = np.repeat(np.arange(F, dtype=np.int64), counts)
    order = np.lexsort((states, fr))                 # state-sorted within each frame
    rank = np.empty(ntok, dtype=np.int64)
    rank[order] = np.arange(ntok, dtype=np.int64) - foff[fr[order]]
    parc64 = parc.astype(np.int64)
    emit = (parc64 >= 0) & (wfst.arc_ilabel[np.maximum(parc64, 0)] > 0)
    pframe = np.where(emit, fr - 1, fr)
    gpred = np.where(parc64 >= 0, foff[np.maximum(pframe, 0)] + pidx, 0)
    pred_sorted = np.where(parc64 >= 0, rank[gpred], -1)
    s_states, s_costs = states[order], costs[order]
    s_parc, s_pred, s_packs = parc64[order], pred_sorted[order], packs[order]
    frames = []
    for f in range(F):
        a, b = foff[f], foff[f + 1]
        frames.append(FrameTokens(f, s_states[a:b].copy(), s_costs[a:b].copy(), s_parc[a:b].copy(),
                                  s_pred[a:b].copy()))
    if collect_frame_packs:
        r.frame_packs = [(fr_.states, s_packs[foff[f]:foff[f + 1]].copy())
                         for f, fr_ in enumerate(frames)]
    if not want_lattice:
        return
    boff = np.zeros(F + 1, dtype=np.int64)
    larc = np.zeros(nlat, dtype=np.int32)
    lfrom = np.zeros(nlat, dtype=np.int32)
    lto = np.zeros(nlat, dtype=np.int32)
    lext = np.zeros(nlat)
    _raise_status(L.lb_result_lattice(res, u, ptr(boff, P64), ptr(larc, P32), ptr(lfrom, P32),
                                      ptr(lto, P32), ptr(lext, PD)), _lib.last_error())
    blk = np.repeat(np.arange(F, dtype=np.int64), np.diff(boff))
    a64 = larc.astype(np.int64)
    il = wfst.arc_ilabel[a64].astype(np.int64)
    ffr = np.where(il > 0, blk - 1, blk)
    from_r = rank[foff[np.maximum(ffr, 0)] + lfrom]
    to_r = rank[foff[blk] + lto]
    acost = np.zeros(nlat)
    em = il > 0
    acost[em] = m[blk[em] - 1, il[em] - 1] * float(cfg.acoustic_scale)
    w = wfst.arc_weight[a64]
    fwd_from = s_costs[foff[np.maximum(ffr, 0)] + from_r]
    cand = np.where(em, (fwd_from + w) + acost, fwd_from + w)
    status = np.where(lext > float(cfg.lattice_beam), STATUS_PRUNED, STATUS_LIVE).astype(np.uint8)
    blocks = []
    for b in range(F):
        s, e = boff[b], boff[b + 1]
        o = s + np.lexsort((from_r[s:e], a64[s:e]))
        blocks.append({"arc_id": a64[o], "from_idx": from_r[o], "to_idx": to_r[o],
                       "acoustic_cost": acost[o], "cost": cand[o], "extra": lext[o],
                       "status": status[o]})
    last = frames[-1]
    finals = wfst.final_cost_array[last.states]
    start_pos = int(np.searchsorted(frames[0].states, wfst.start_state))
    lat = WorkLattice(wfst, frames, blocks, None, start_pos, r.partial,
                      None if r.partial else finals, r.total_cost)
    r.work_lattice = lat


# ---------------------------------------------------------------------------
# Single-op surfaces (decoder.py:373-456)
# ---------------------------------------------------------------------------

def _frontier(wfst, states, costs):
    states = np.asarray(states, dtype=np.int64)
    costs = np.asarray(costs, dtype=np.float64)
    if states.ndim != 1 or states.shape != costs.shape:
        raise UsageError("states and costs must be matching 1-d sequences")
    if len(states) == 0:
        raise UsageError("frontier is empty")
    if len(np.unique(states)) != len(states):
        raise UsageError("frontier states must be unique")
    if states.min() < 0 or states.max() >= wfst.num_states:
        raise UsageError("frontier state outside the graph")
    o = np.argsort(states, kind="stable")
    return np.ascontiguousarray(states[o], dtype=np.int32), np.ascontiguousarray(costs[o])


def expand_emitting(wfst, states, costs, matrix: CostMatrix, frame: int, beam: float,
                    acoustic_scale: float = 1.0, device: int = 0):
    """One emitting pass on the device; (sorted states, costs, cutoff) of the
    winners under best + beam (decoder.py:373-400)."""
    m = _matrix_array(matrix)
    if not 0 <= frame < m.shape[0]:
        raise UsageError(f"frame {frame} outside the matrix's {m.shape[0]} frames")
    s, c = _frontier(wfst, states, costs)
    if not (math.isfinite(beam) and beam > 0):
        raise UsageError("beam must be a positive finite number")
    if int(wfst.max_ilabel) > m.shape[1]:
        raise UsageError("graph uses an input label beyond the cost matrix columns")
    row = np.ascontiguousarray(m[frame] * float(acoustic_scale))
    g = device_graph(wfst, device)
    S = int(wfst.num_states)
    os_, oc = np.zeros(S, dtype=np.int32), np.zeros(S)
    n_out, cut = C.c_int64(), C.c_double()
    rc = _lib.lib().lb_expand_emitting(g.handle, ptr(s, P32), ptr(c, PD), len(s), ptr(row, PD),
                                       m.shape[1], float(beam), ptr(os_, P32), ptr(oc, PD),
                                       C.byref(n_out), C.byref(cut))
    _raise_status(rc, _lib.last_error())
    k = n_out.value
    o = np.argsort(os_[:k], kind="stable")
    if not math.isfinite(cut.value):
        return np.empty(0, dtype=np.int64), np.empty(0), math.inf
    return os_[:k][o].astype(np.int64), oc[:k][o], float(cut.value)


def expand_nonemitting(wfst, states, costs, cutoff: float, device: int = 0):
    """Epsilon closure of one frontier under a fixed cutoff (decoder.py:403-435)."""
    s, c = _frontier(wfst, states, costs)
    g = device_graph(wfst, device)
    S = int(wfst.num_states)
    os_, oc = np.zeros(S, dtype=np.int32), np.zeros(S)
    n_out = C.c_int64()
    rc = _lib.lib().lb_expand_nonemitting(g.handle, ptr(s, P32), ptr(c, PD), len(s), float(cutoff),
                                          ptr(os_, P32), ptr(oc, PD), C.byref(n_out))
    _raise_status(rc, _lib.last_error())
    k = n_out.value
    o = np.argsort(os_[:k], kind="stable")
    return os_[:k][o].astype(np.int64), oc[:k][o]
