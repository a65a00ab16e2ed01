"""Shared comparison helpers: device results vs the CPU oracle (oracle/)."""

from __future__ import annotations

import numpy as np

import paper_1804_03243_b200 as lb

ERRMAP = {1: lb.DecodeFailure, 2: lb.UsageError, 3: lb.CapacityError, 4: lb.InternalInvariantError}


def near_boundary(ref, lattice_beam, tol=1e-3) -> bool:
    """C3 skip rule (test_acceptance.py:151-165): an oracle extra within tol of the beam."""
    for blk in ref.blocks:
        ex = blk[4]
        if len(ex) and np.min(np.abs(ex - lattice_beam)) <= tol:
            return True
    return False


def compare_1best(got, ref, frame_packs=True):
    assert got.words == ref.words, (got.words, ref.words)
    assert got.alignment == ref.alignment
    assert got.total_cost == ref.total_cost, (got.total_cost, ref.total_cost)
    assert got.partial == ref.partial
    if frame_packs:
        assert len(got.frame_packs) == len(ref.frame_packs)
        for f, ((s1, p1), (s2, p2)) in enumerate(zip(got.frame_packs, ref.frame_packs)):
            assert np.array_equal(s1, s2), f"frame {f} states differ"
            assert np.array_equal(p1, p2), f"frame {f} packs differ"


def _final_arc_keys(fl_from, fl_to, il, ol, g, ac, node_frame, node_idx):
    """FinalLattice arcs as renumbering-independent keys:
    (from frame, from token, to frame, to token, ilabel, olabel, graph, acoustic)."""
    nf, ni = np.asarray(node_frame), np.asarray(node_idx)
    f, t = np.asarray(fl_from), np.asarray(fl_to)
    return list(zip(nf[f].tolist(), ni[f].tolist(), nf[t].tolist(), ni[t].tolist(),
                    np.asarray(il).tolist(), np.asarray(ol).tolist(),
                    np.asarray(g).tolist(), np.asarray(ac).tolist()))


def _boundary_keys(ref, wfst, lattice_beam, tol):
    """Keys of the live arcs whose oracle extra lies within tol of lattice_beam."""
    keys = set()
    for b, blk in enumerate(ref.blocks):
        arcs, frm, to, acv, extra, _ = blk
        near = np.flatnonzero(np.abs(extra - lattice_beam) <= tol)
        for k in near:
            a = int(arcs[k])
            il = int(wfst.arc_ilabel[a])
            keys.add((b - 1 if il > 0 else b, int(frm[k]), b, int(to[k]), il, int(wfst.arc_olabel[a]),
                      float(wfst.arc_weight[a]), float(acv[k])))
    return keys


def compare_lattice(got, ref, lattice_beam, tol=1e-3):
    """Live-arc extras within 1e-4 always.  The FinalLattice arrays must be
    identical; when an oracle extra lies within tol of lattice_beam (the
    reference's C3 rule, test_acceptance.py:151-165) the survivor set of those
    arcs may legitimately differ, so the final lattices are compared on every
    arc AWAY from the beam instead (keys independent of node renumbering), and
    on the final nodes those arcs reach."""
    wl = got.work_lattice
    for b, blk in enumerate(ref.blocks):
        arcs, _, _, _, extra, _ = blk
        ga = wl.block_arrays(b)
        assert np.array_equal(np.sort(ga["arc_id"]), np.sort(arcs)), f"block {b} live arc set differs"
        o1, o2 = np.argsort(ga["arc_id"], kind="stable"), np.argsort(arcs, kind="stable")
        e1, e2 = ga["extra"][o1], extra[o2]
        fin = np.isfinite(e2)
        assert np.array_equal(np.isfinite(e1), fin), f"block {b} dead-end pattern differs"
        if fin.any():
            assert np.max(np.abs(e1[fin] - e2[fin])) <= 1e-4, f"block {b} extras differ"
    fl, rf = got.lattice, ref.final
    if not near_boundary(ref, lattice_beam, tol):
        assert fl.num_nodes == rf["num_nodes"] and fl.start == rf["start"]
        for k in ("final_ids", "final_costs", "from_", "to", "ilabel", "olabel", "graph_cost",
                  "acoustic_cost", "node_frame", "node_idx"):
            assert np.array_equal(getattr(fl, k), rf[k]), f"final lattice {k} differs"
        return "exact"
    wfst = getattr(ref, "wfst", None)
    assert wfst is not None, "boundary comparison needs the graph (decode_both sets ref.wfst)"
    skip = _boundary_keys(ref, wfst, lattice_beam, tol)
    dk = _final_arc_keys(fl.from_, fl.to, fl.ilabel, fl.olabel, fl.graph_cost, fl.acoustic_cost,
                         fl.node_frame, fl.node_idx)
    rk = _final_arc_keys(rf["from_"], rf["to"], rf["ilabel"], rf["olabel"], rf["graph_cost"],
                         rf["acoustic_cost"], rf["node_frame"], rf["node_idx"])
    dkeep = sorted(k for k in dk if k not in skip)
    rkeep = sorted(k for k in rk if k not in skip)
    assert dkeep == rkeep, f"final lattice arcs away from the beam differ ({len(dkeep)} vs {len(rkeep)})"
    # final nodes reached by those arcs: same (frame, token) and graph final cost
    reach = {(k[2], k[3]) for k in rkeep}
    df = {(int(fl.node_frame[i]), int(fl.node_idx[i])): c for i, c in zip(fl.final_ids, fl.final_costs)}
    rfn = {(int(rf["node_frame"][i]), int(rf["node_idx"][i])): c
           for i, c in zip(rf["final_ids"], rf["final_costs"])}
    assert {k: v for k, v in df.items() if k in reach} == {k: v for k, v in rfn.items() if k in reach}
    return "boundary"


def decode_both(w, m, oracle, beam, lattice_beam=4.0, scale=1.0, max_active=0, want_lattice=True,
                device_kw=None, **cfg_kw):
    ref = oracle.decode(w, m, beam, lattice_beam=lattice_beam, acoustic_scale=scale,
                        max_active=max_active, want_lattice=want_lattice, **cfg_kw)
    cfg = lb.DecodeConfig(beam=beam, lattice_beam=lattice_beam, acoustic_scale=scale,
                          max_active=max_active, max_lattice_arcs=50_000_000, keep_work_lattice=True,
                          **{k: v for k, v in cfg_kw.items() if k in ("max_tokens_per_frame",)},
                          **(device_kw or {}))
    try:
        got = lb.decode_utterance(w, m, cfg, want_lattice=want_lattice, collect_frame_packs=True)
    except lb.LatbeamError as exc:
        got = exc
    ref.wfst = w
    return got, ref


def check_pair(got, ref, lattice_beam, want_lattice=True):
    if not ref.ok:
        assert isinstance(got, ERRMAP[ref.status]), (got, ref.message)
        return "error"
    assert not isinstance(got, Exception), (got, "oracle decoded fine")
    compare_1best(got, ref)
    if want_lattice:
        return compare_lattice(got, ref, lattice_beam)
    return "ok"
