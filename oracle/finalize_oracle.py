"""numpy restatement of the reference's `finalize_lattice` (TEST INFRASTRUCTURE).

Only tests/ import this: it checks the device single-op surface
`paper_1804_03243_b200.finalize_lattice` (C-ABI lb_finalize_lattice).  It follows
/root/reference/pkg/src/latbeam/lattice.py:537-598: live arcs; node key
(frame << 32) | idx, np.unique + np.searchsorted renumbering; start check; final
nodes at the last frame with a finite final cost (all of them, cost 0, when
partial); canonical np.lexsort((acoustic, graph, olabel, ilabel, to, from)).
Returns a dict of the FinalLattice fields, or raises ValueError with the
reference's DecodeFailure message.
"""

from __future__ import annotations

import numpy as np


def finalize(t: dict, start_idx: int, last: int, partial: bool, final_token_costs):
    if len(t["from_frame"]) == 0:
        raise ValueError("no lattice arcs survived pruning")
    fk = (t["from_frame"].astype(np.int64) << 32) | t["from_idx"].astype(np.int64)
    tk = (t["to_frame"].astype(np.int64) << 32) | t["to_idx"].astype(np.int64)
    keys = np.unique(np.concatenate([fk, tk]))
    fid = np.searchsorted(keys, fk)
    tid = np.searchsorted(keys, tk)
    order = np.lexsort((t["acoustic_cost"], t["graph_cost"], t["olabel"], t["ilabel"], tid, fid))
    nframe = keys >> 32
    nidx = keys & 0xFFFFFFFF
    sp = int(np.searchsorted(keys, np.int64(start_idx)))
    if sp >= len(keys) or keys[sp] != start_idx:
        raise ValueError("surviving arcs do not connect to the start node")
    at_last = nframe == last
    if partial:
        fids = np.flatnonzero(at_last)
        fcs = np.zeros(len(fids))
    else:
        tc = final_token_costs
        fin = at_last & np.isfinite(tc[np.where(at_last, nidx, 0)])
        fids = np.flatnonzero(fin)
        fcs = tc[nidx[fids]]
    if len(fids) == 0:
        raise ValueError("no terminal node survived pruning")
    return dict(num_nodes=len(keys), start=sp, final_ids=fids.astype(np.int64), final_costs=fcs.astype(np.float64),
                from_=fid[order].astype(np.int64), to=tid[order].astype(np.int64),
                ilabel=t["ilabel"][order].astype(np.int64), olabel=t["olabel"][order].astype(np.int64),
                graph_cost=t["graph_cost"][order].astype(np.float64),
                acoustic_cost=t["acoustic_cost"][order].astype(np.float64),
                node_frame=nframe.astype(np.int64), node_idx=nidx.astype(np.int64))
