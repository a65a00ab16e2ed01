"""Lattice scoring — mirrors `latbeam.scoring` (scoring.py:1-130).

`oracle_wer` runs on the GPU (csrc/lb_scoring.cuh, one CTA per lattice;
`oracle_wer_batch` scores many lattices in one launch).  `wer` and
`lattice_density` are small host computations, as in the reference.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import UsageError
from .lattice import FinalLattice


@dataclass(frozen=True)
class WerResult:
    substitutions: int
    insertions: int
    deletions: int

    @property
    def errors(self) -> int:
        return self.substitutions + self.insertions + self.deletions


def wer(hyp: list[int], ref: list[int]) -> WerResult:
    """Edit-distance word counts; ties prefer substitutions, then insertions,
    then deletions (scoring.py:24-58)."""
    if len(ref) == 0:
        raise UsageError("reference word sequence is empty")
    h, r = len(hyp), len(ref)
    d = np.zeros((h + 1, r + 1), dtype=np.int64)
    d[:, 0] = np.arange(h + 1)
    d[0, :] = np.arange(r + 1)
    for i in range(1, h + 1):
        sub = d[i - 1, :-1] + (np.asarray(ref) != hyp[i - 1])
        row = np.minimum(sub, d[i - 1, 1:] + 1)
        d[i, 1:] = row
        for j in range(1, r + 1):          # deletions run along the row
            d[i, j] = min(d[i, j], d[i, j - 1] + 1)
    subs = ins = dels = 0
    i, j = h, r
    while i > 0 or j > 0:
        if i > 0 and j > 0 and d[i, j] == d[i - 1, j - 1] + (hyp[i - 1] != ref[j - 1]):
            subs += int(hyp[i - 1] != ref[j - 1])
            i, j = i - 1, j - 1
        elif i > 0 and d[i, j] == d[i - 1, j] + 1:
            ins += 1
            i -= 1
        else:
            dels += 1
            j -= 1
    return WerResult(subs, ins, dels)


def wer_percent(hyp: list[int], ref: list[int]) -> float:
    return 100.0 * wer(hyp, ref).errors / len(ref)


class _View(C.Structure):
    _fields_ = [("num_nodes", C.c_int64), ("start", C.c_int64), ("n_final", C.c_int64),
                ("n_arcs", C.c_int64), ("n_ref", C.c_int64), ("final_ids", _lib.P64),
                ("from_", _lib.P64), ("to", _lib.P64), ("olabel", _lib.P64), ("node_frame", _lib.P64),
                ("ref", _lib.P32)]


def oracle_wer_batch(lattices: list[FinalLattice], refs: list[list[int]], device: int = 0) -> list[int]:
    """Fewest word errors over complete paths of each lattice (scoring.py:66-114),
    all lattices in one GPU launch.  Raises UsageError like the reference."""
    if len(lattices) != len(refs):
        raise UsageError("one reference per lattice")
    keep, views = [], []
    for fl, ref in zip(lattices, refs):
        if len(ref) == 0:
            raise UsageError("reference word sequence is empty")
        cols = [np.ascontiguousarray(x, dtype=np.int64) for x in (fl.final_ids, fl.from_, fl.to, fl.olabel)]
        nf = None if fl.node_frame is None else np.ascontiguousarray(fl.node_frame, dtype=np.int64)
        r = np.ascontiguousarray(ref, dtype=np.int32)
        keep.append((cols, nf, r))
        views.append(_View(int(fl.num_nodes), int(fl.start), len(cols[0]), len(cols[1]), len(r),
                           *[c.ctypes.data_as(_lib.P64) for c in cols],
                           nf.ctypes.data_as(_lib.P64) if nf is not None else _lib.P64(),
                           r.ctypes.data_as(_lib.P32)))
    n = len(views)
    if n == 0:
        return []
    arr = (_View * n)(*views)
    out = np.zeros(n, dtype=np.int64)
    L = _lib.lib()
    rc = L.lb_oracle_wer_batch(int(device), n, C.cast(arr, C.c_void_p), out.ctypes.data_as(_lib.P64))
    if rc != 0:
        raise UsageError(_lib.last_error())
    res = []
    for x in out.tolist():
        if x == -1:
            raise UsageError("lattice has no complete path")
        if x == -2:
            raise UsageError("lattice oracle search failed to converge")
        res.append(int(x))
    return res


def oracle_wer(fl: FinalLattice, ref: list[int], device: int = 0) -> int:
    return oracle_wer_batch([fl], [ref], device)[0]


def oracle_wer_percent(fl: FinalLattice, ref: list[int]) -> float:
    return 100.0 * oracle_wer(fl, ref) / len(ref)


def lattice_density(fl: FinalLattice, num_frames: int | None = None) -> float:
    """Arcs per acoustic frame (scoring.py:121-130)."""
    t = num_frames if num_frames is not None else fl.num_frames
    if t is None:
        raise UsageError("lattice does not carry a frame count; pass num_frames")
    if t < 1:
        raise UsageError("frame count must be >= 1")
    return fl.num_arcs / float(t)
