"""CPU restatement of the reference's `prune_lattice` (TEST INFRASTRUCTURE).

Only tests/ import this: it is the checker for the device single-op surface
`paper_1804_03243_b200.prune_lattice` (C-ABI lb_prune_lattice).  It follows
/root/reference/pkg/src/latbeam/lattice.py:365-497 -- `prune_lattice` (terminus,
backward sweeps), `_relax_frame` (emitting relaxation of block f+1 with
np.minimum.at, Jacobi in-frame epsilon fixpoint with tolerance 1e-9, clamp at 0)
and `_flag_block` (extra of every LIVE arc, PRUNED when extra > lattice_beam) --
over plain arrays: frames = [(costs)], blocks = [dict(from_idx, to_idx, ilabel,
graph_cost, acoustic_cost, status, extra)] with status 0 LIVE / 1 PRUNED.
"""

from __future__ import annotations

import numpy as np

CONVERGE_TOL = 1e-9   # lattice.py:36


def relax_frame(frames, blocks, node_extra, f, t, terminus):
    """lattice.py:434-470."""
    n = len(frames[f])
    fwd = frames[f]
    new = terminus.copy() if f == t else np.full(n, np.inf)
    if f < t:
        b = blocks[f + 1]
        sel = (b["status"] == 0) & (b["ilabel"] > 0)
        if np.any(sel):
            nxt = node_extra[f + 1]
            fwd_next = frames[f + 1]
            cand = (fwd[b["from_idx"][sel]] + b["graph_cost"][sel] + b["acoustic_cost"][sel]
                    - fwd_next[b["to_idx"][sel]] + nxt[b["to_idx"][sel]])
            np.minimum.at(new, b["from_idx"][sel], cand)
    b = blocks[f]
    sel = (b["status"] == 0) & (b["ilabel"] == 0)
    if np.any(sel):
        src, dst = b["from_idx"][sel], b["to_idx"][sel]
        base = fwd[src] + b["graph_cost"][sel] - fwd[dst]
        for _ in range(n + 1):
            cand = base + new[dst]
            before = new[src].copy()
            np.minimum.at(new, src, cand)
            with np.errstate(invalid="ignore"):
                moved = np.any(before - new[src] > CONVERGE_TOL)
            if not moved:
                break
        else:
            raise RuntimeError(f"epsilon extra-cost fixpoint did not settle within frame {f}")
    return np.maximum(new, 0.0)


def prune(frames, blocks, t, lattice_beam, terminus):
    """lattice.py:365-431 + 473-497, from scratch (one backward sweep reaches the
    fixpoint of this layered relaxation; the reference's second sweep confirms)."""
    node_extra = [None] * len(frames)
    for f in range(t, -1, -1):
        node_extra[f] = relax_frame(frames, blocks, node_extra, f, t, terminus)
    out = []
    for bi in range(t + 1):
        b = {k: v.copy() for k, v in blocks[bi].items()}
        live = b["status"] == 0
        if np.any(live):
            il = b["ilabel"][live]
            fr = np.where(il > 0, bi - 1, bi)
            fwd_from = np.array([frames[x][i] for x, i in zip(fr, b["from_idx"][live])], dtype=np.float64)
            fwd_to = frames[bi][b["to_idx"][live]]
            x = np.maximum(fwd_from + b["graph_cost"][live] + b["acoustic_cost"][live] - fwd_to
                           + node_extra[bi][b["to_idx"][live]], 0.0)
            ex = b["extra"].copy()
            ex[live] = x
            st = b["status"].copy()
            idx = np.flatnonzero(live)
            st[idx[x > lattice_beam]] = 1
            b["extra"], b["status"] = ex, st
        out.append(b)
    return out, node_extra
