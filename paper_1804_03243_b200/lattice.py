"""Lattice result types and the host-side canonicalisation of device lattices.

The device records every live lattice arc (SURVEY.md Appendix A.5 rule) and its
pruning extra cost (csrc/lb_kernels.cuh `prune_kernel`, restating
lattice.py:365-497 of `latbeam`).  This module turns those device arrays into
the reference's result types:

* `FrameTokens` — one frame's state-sorted token list (lattice.py:71-98);
* `WorkLattice` — the reference `Lattice` query surface (`frames`,
  `block_arrays`, `live_arc_table`, `arcs`, `partial`, `final_token_costs`)
  over the device results; arcs are LIVE or PRUNED (no VOID slots exist because
  only live passes are ever recorded);
* `FinalLattice` + `finalize_lattice` — dense (frame, index) renumbering and
  canonical arc order (lattice.py:500-598);
* the text format (lattice.py:605-673).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import NamedTuple

import numpy as np

from .errors import DecodeFailure, ParseError

STATUS_LIVE = 0
STATUS_PRUNED = 1
STATUS_VOID = 2


class LatticeNodeId(NamedTuple):
    frame: int
    idx: int


@dataclass(frozen=True)
class LatticeArc:
    from_node: LatticeNodeId
    to_node: LatticeNodeId
    ilabel: int
    olabel: int
    graph_cost: float
    acoustic_cost: float
    extra_cost: float = math.inf
    pruned: bool = False


@dataclass(frozen=True)
class Token:
    cost: float
    pred_arc: int | None
    pred_token: int | None
    state: int
    frame: int


@dataclass
class FrameTokens:
    """One frame's tokens, sorted by state; pred_idx indexes the previous
    frame for an emitting pred arc and this frame for an epsilon one."""

    frame: int
    states: np.ndarray
    costs: np.ndarray
    pred_arc: np.ndarray
    pred_idx: np.ndarray

    @property
    def n(self) -> int:
        return len(self.states)

    def token(self, i: int) -> Token:
        return Token(float(self.costs[i]),
                     int(self.pred_arc[i]) if self.pred_arc[i] >= 0 else None,
                     int(self.pred_idx[i]) if self.pred_idx[i] >= 0 else None,
                     int(self.states[i]), self.frame)


@dataclass
class FinalLattice:
    num_nodes: int
    start: int
    final_ids: np.ndarray
    final_costs: np.ndarray
    from_: np.ndarray
    to: np.ndarray
    ilabel: np.ndarray
    olabel: np.ndarray
    graph_cost: np.ndarray
    acoustic_cost: np.ndarray
    node_frame: np.ndarray | None = None
    node_idx: np.ndarray | None = None
    num_frames: int | None = None

    @property
    def num_arcs(self) -> int:
        return len(self.from_)

    def same_lattice(self, other) -> bool:
        keys = ("final_ids", "final_costs", "from_", "to", "ilabel", "olabel", "graph_cost",
                "acoustic_cost")
        return (self.num_nodes == other.num_nodes and self.start == other.start
                and all(np.array_equal(getattr(self, k), getattr(other, k)) for k in keys))


class WorkLattice:
    """Query view of one decoded utterance's lattice (reference `Lattice` surface)."""

    def __init__(self, wfst, frames, blocks, node_extra, start_idx, partial, final_token_costs,
                 best_final_cost):
        self.wfst = wfst
        self.frames: list[FrameTokens] = frames
        self._blocks = blocks           # per block: dict(arc_id, from_idx, to_idx, acoustic_cost, extra, status)
        self.node_extra = node_extra
        self.start_idx = start_idx
        self.partial = partial
        self.final_token_costs = final_token_costs
        self.best_final_cost = best_final_cost
        self.final_prune_done = True

    @property
    def num_frames(self) -> int:
        return len(self.frames) - 1

    def block_arrays(self, block: int) -> dict[str, np.ndarray]:
        b = self._blocks[block]
        a = b["arc_id"]
        il = self.wfst.arc_ilabel[a].astype(np.int64)
        n = len(a)
        return {
            "slots": np.arange(n, dtype=np.int64),
            "arc_id": a,
            "ilabel": il,
            "olabel": self.wfst.arc_olabel[a].astype(np.int64),
            "graph_cost": self.wfst.arc_weight[a],
            "acoustic_cost": b["acoustic_cost"],
            "cost": b["cost"],
            "from_frame": np.where(il > 0, block - 1, block).astype(np.int64),
            "from_idx": b["from_idx"],
            "to_frame": np.full(n, block, dtype=np.int64),
            "to_idx": b["to_idx"],
            "status": b["status"],
            "extra": b["extra"],
        }

    def live_arc_table(self, include_pruned: bool = False) -> dict[str, np.ndarray]:
        cols: dict[str, list] = {}
        for b in range(len(self.frames)):
            blk = self.block_arrays(b)
            keep = blk["status"] == STATUS_LIVE
            if include_pruned:
                keep |= blk["status"] == STATUS_PRUNED
            for k, v in blk.items():
                cols.setdefault(k, []).append(v[keep])
        return {k: np.concatenate(v) if v else np.empty(0) for k, v in cols.items()}

    def arcs(self, include_pruned: bool = False) -> list[LatticeArc]:
        t = self.live_arc_table(include_pruned)
        return [LatticeArc(LatticeNodeId(int(t["from_frame"][i]), int(t["from_idx"][i])),
                           LatticeNodeId(int(t["to_frame"][i]), int(t["to_idx"][i])),
                           int(t["ilabel"][i]), int(t["olabel"][i]), float(t["graph_cost"][i]),
                           float(t["acoustic_cost"][i]), float(t["extra"][i]),
                           bool(t["status"][i] == STATUS_PRUNED))
                for i in range(len(t["slots"]))]


class LazyWorkLattice(WorkLattice):
    """A WorkLattice built on first use.

    The reference returns `DecodeResult.work_lattice` whenever a lattice is
    requested (decoder.py:605-606).  Shipping every live arc and token list to
    the host costs more than the decode itself (C1: ~12.6M arcs per utterance),
    so results carry this proxy instead: the first attribute access re-decodes
    the utterance with `keep_work_lattice=True` -- decoding is deterministic and
    bit-exact, so it is the same lattice -- and adopts it."""

    def __init__(self, build):   # noqa: D401 - no WorkLattice state until built
        self.__dict__["_build"] = build

    def _materialise(self):
        build = self.__dict__.get("_build")
        if build is not None:
            real = build()
            self.__dict__["_build"] = None
            self.__dict__.update(real.__dict__)

    def __getattr__(self, name):
        if name.startswith("__") or self.__dict__.get("_build") is None:
            raise AttributeError(name)
        self._materialise()
        return getattr(self, name)


def prune_lattice(lat: WorkLattice, frontier: FrameTokens, lattice_beam: float,
                  final_costs: np.ndarray | None = None, device: int = 0) -> None:
    """Flag arcs whose extra cost exceeds lattice_beam (lattice.py:365-431 of
    `latbeam`), on the device (C-ABI lb_prune_lattice, csrc `prune_op_kernel`).

    Node extras start at the frontier (zeros, or totals - min(totals) when
    final_costs is given) and relax backward frame by frame with an in-frame
    epsilon fixpoint; an arc's extra is fwd(from) + graph + acoustic - fwd(to) +
    node_extra(to), clamped at 0.  LIVE arcs of blocks 0..t get their extra and
    turn PRUNED when it exceeds lattice_beam; already-pruned arcs stay pruned and
    do not participate.  Mutates `lat` (block extras / statuses, node_extra)."""
    import ctypes as C

    from . import _lib
    from .errors import InternalInvariantError, UsageError
    if not lattice_beam >= 0:
        raise UsageError("lattice_beam must be >= 0")
    t = frontier.frame
    if not (0 <= t < len(lat.frames)) or lat.frames[t] is not frontier:
        raise UsageError("frontier is not a frame of this lattice")
    if frontier.n == 0:
        raise UsageError("frontier is empty")
    if final_costs is None:
        terminus = np.zeros(frontier.n)
    else:
        totals = frontier.costs + np.asarray(final_costs, dtype=np.float64)
        best_total = totals.min()
        if not math.isfinite(best_total):
            raise UsageError("final_costs leave no finite-cost terminus")
        terminus = totals - best_total
    fo = np.zeros(t + 2, dtype=np.int64)
    fo[1:] = np.cumsum([lat.frames[f].n for f in range(t + 1)])
    fwd = np.ascontiguousarray(np.concatenate([lat.frames[f].costs for f in range(t + 1)]), dtype=np.float64)
    blks = [lat.block_arrays(b) for b in range(t + 1)]
    bo = np.zeros(t + 2, dtype=np.int64)
    bo[1:] = np.cumsum([len(b["arc_id"]) for b in blks])

    def cat(key, dt):
        return np.ascontiguousarray(np.concatenate([b[key] for b in blks]) if blks else np.empty(0), dtype=dt)
    frm, to = cat("from_idx", np.int32), cat("to_idx", np.int32)
    emit = np.ascontiguousarray(cat("ilabel", np.int64) > 0, dtype=np.uint8)
    g, ac = cat("graph_cost", np.float64), cat("acoustic_cost", np.float64)
    status = np.ascontiguousarray(np.where(cat("status", np.uint8) == STATUS_LIVE, 0, 1), dtype=np.uint8)
    extra = cat("extra", np.float64)
    node_extra = np.zeros(int(fo[-1]))
    terminus = np.ascontiguousarray(terminus, dtype=np.float64)
    P64, P32, PD, U8 = _lib.P64, _lib.P32, _lib.PD, C.POINTER(C.c_uint8)
    L = _lib.lib()
    rc = L.lb_prune_lattice(int(device), int(t), fo.ctypes.data_as(P64), fwd.ctypes.data_as(PD),
                            bo.ctypes.data_as(P64), frm.ctypes.data_as(P32), to.ctypes.data_as(P32),
                            emit.ctypes.data_as(U8), g.ctypes.data_as(PD), ac.ctypes.data_as(PD),
                            terminus.ctypes.data_as(PD), float(lattice_beam), status.ctypes.data_as(U8),
                            extra.ctypes.data_as(PD), node_extra.ctypes.data_as(PD))
    if rc == 4:
        raise InternalInvariantError(_lib.last_error())
    if rc != 0:
        raise UsageError(_lib.last_error())
    for b in range(t + 1):
        s_, e_ = int(bo[b]), int(bo[b + 1])
        lat._blocks[b]["extra"] = extra[s_:e_].copy()
        lat._blocks[b]["status"] = np.where(status[s_:e_] == 0, STATUS_LIVE, STATUS_PRUNED).astype(np.uint8)
    ne = list(lat.node_extra) if lat.node_extra is not None else [None] * len(lat.frames)
    for f in range(t + 1):
        ne[f] = node_extra[int(fo[f]):int(fo[f + 1])].copy()
    lat.node_extra = ne


def finalize_lattice(lat: WorkLattice, device: int = 0) -> FinalLattice:
    """Compact surviving arcs, renumber nodes densely by (frame, idx), sort arcs
    canonically by (from, to, ilabel, olabel, graph, acoustic) -- lattice.py:537-598
    of `latbeam` -- on the device (C-ABI lb_finalize_lattice: CUB radix sorts,
    unique and the six stable LSD passes of np.lexsort, as the decode path's own
    finaliser does, csrc/lb_lattice.cuh)."""
    import ctypes as C

    from . import _lib
    from .errors import InternalInvariantError, UsageError
    t = lat.live_arc_table()
    n = len(t["slots"])
    fk = np.ascontiguousarray((t["from_frame"].astype(np.uint64) << np.uint64(32)) | t["from_idx"].astype(np.uint64))
    tk = np.ascontiguousarray((t["to_frame"].astype(np.uint64) << np.uint64(32)) | t["to_idx"].astype(np.uint64))
    il = np.ascontiguousarray(t["ilabel"], dtype=np.int32)
    ol = np.ascontiguousarray(t["olabel"], dtype=np.int32)
    g = np.ascontiguousarray(t["graph_cost"], dtype=np.float64)
    ac = np.ascontiguousarray(t["acoustic_cost"], dtype=np.float64)
    last = lat.num_frames
    fc = None if lat.partial or lat.final_token_costs is None else \
        np.ascontiguousarray(lat.final_token_costs, dtype=np.float64)
    L = _lib.lib()
    P32, PD, PU64 = _lib.P32, _lib.PD, _lib.PU64
    res = _lib.PV()
    rc = L.lb_finalize_lattice(int(device), n, fk.ctypes.data_as(PU64), tk.ctypes.data_as(PU64),
                               il.ctypes.data_as(P32), ol.ctypes.data_as(P32), g.ctypes.data_as(PD),
                               ac.ctypes.data_as(PD), int(lat.start_idx), int(last), int(bool(lat.partial)),
                               0 if fc is None else len(fc), None if fc is None else fc.ctypes.data_as(PD),
                               C.byref(res))
    if rc != 0:
        raise (UsageError if rc == 2 else InternalInvariantError)(_lib.last_error())
    try:
        st = C.c_int32()
        msg = C.create_string_buffer(256)
        L.lb_result_status(res, 0, C.byref(st), msg, 256, None, 0)
        if st.value == 1:
            raise DecodeFailure(msg.value.decode())
        from .decoder import _final_lattice
        return _final_lattice(res, 0, last)
    finally:
        L.lb_result_free(res)


def write_lattice_text(fl: FinalLattice) -> str:
    """The reference lattice text (lattice.py:605-614), formatted by the native
    library (multi-threaded, floats as Python repr; byte-identical to
    `write_lattice_text_py`)."""
    import ctypes as C

    from . import _lib
    L = _lib.host_lib()
    i64 = [np.ascontiguousarray(getattr(fl, k), dtype=np.int64)
           for k in ("final_ids", "from_", "to", "ilabel", "olabel")]
    f64 = [np.ascontiguousarray(getattr(fl, k), dtype=np.float64)
           for k in ("final_costs", "graph_cost", "acoustic_cost")]
    P64, PD = _lib.P64, _lib.PD
    args = (int(fl.num_nodes), int(fl.start), len(i64[0]), i64[0].ctypes.data_as(P64),
            f64[0].ctypes.data_as(PD), len(i64[1]), i64[1].ctypes.data_as(P64),
            i64[2].ctypes.data_as(P64), i64[3].ctypes.data_as(P64), i64[4].ctypes.data_as(P64),
            f64[1].ctypes.data_as(PD), f64[2].ctypes.data_as(PD))
    n = L.lb_lattice_text(*args, None, 0)
    buf = C.create_string_buffer(int(n))
    L.lb_lattice_text(*args, buf, n)
    return buf.raw[:n].decode()


def write_lattice_text_py(fl: FinalLattice) -> str:
    """Pure-Python twin of write_lattice_text (the format's executable spec)."""
    out = [f"NODES {fl.num_nodes} ARCS {fl.num_arcs} START {fl.start}"]
    out += [f"F {fl.final_ids[i]} {float(fl.final_costs[i])!r}" for i in range(len(fl.final_ids))]
    out += [f"A {fl.from_[i]} {fl.to[i]} {fl.ilabel[i]} {fl.olabel[i]} "
            f"{float(fl.graph_cost[i])!r} {float(fl.acoustic_cost[i])!r}" for i in range(fl.num_arcs)]
    return "\n".join(out) + "\n"


def read_lattice_text(text) -> FinalLattice:
    if hasattr(text, "read"):
        text = text.read()
    lines = str(text).splitlines()
    if not lines:
        raise ParseError(1, "empty lattice text")
    h = lines[0].split()
    if len(h) != 6 or h[0] != "NODES" or h[2] != "ARCS" or h[4] != "START":
        raise ParseError(1, f"bad header {lines[0]!r}")
    try:
        n, m, start = int(h[1]), int(h[3]), int(h[5])
    except ValueError:
        raise ParseError(1, f"non-integer header field in {lines[0]!r}") from None
    fids, fcs = [], []
    cols: list[list] = [[] for _ in range(6)]
    for no, line in enumerate(lines[1:], 2):
        f = line.split()
        if not f:
            continue
        try:
            if f[0] == "F" and len(f) == 3:
                fids.append(int(f[1]))
                fcs.append(float(f[2]))
            elif f[0] == "A" and len(f) == 7:
                vals = [int(x) for x in f[1:5]] + [float(f[5]), float(f[6])]
                for c, v in zip(cols, vals):
                    c.append(v)
            else:
                raise ParseError(no, f"unrecognized line {line!r}")
        except ValueError:
            kind = "final" if f[0] == "F" else "arc"
            raise ParseError(no, f"bad {kind} line {line!r}") from None
    if len(cols[0]) != m:
        raise ParseError(len(lines), f"header promised {m} arcs, found {len(cols[0])}")
    ids = np.asarray(fids, dtype=np.int64)
    fr, to = (np.asarray(c, dtype=np.int64) for c in cols[:2])
    if (len(ids) and (ids.min() < 0 or ids.max() >= n)) or any(
            len(r) and (r.min() < 0 or r.max() >= n) for r in (fr, to)) or not 0 <= start < n:
        raise ParseError(1, "node reference out of range")
    return FinalLattice(n, start, ids, np.asarray(fcs, dtype=np.float64), fr, to,
                        np.asarray(cols[2], dtype=np.int64), np.asarray(cols[3], dtype=np.int64),
                        np.asarray(cols[4], dtype=np.float64), np.asarray(cols[5], dtype=np.float64))
