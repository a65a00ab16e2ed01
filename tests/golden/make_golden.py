"""Generate the golden fixtures from the REFERENCE implementation (run here only).

This script imports the reference package `latbeam` from /root/reference
(read-only; numpy engine, NUMBA_CACHE_DIR redirected) and records its outputs
on seeded inputs.  The fixtures pin the CPU oracle (oracle/) and, through it,
the CUDA path.  /root/reference does not exist on the GPU box, so the outputs
are committed here as small .npz files; inputs are regenerated from seeds by
`paper_1804_03243_b200.synthetic` (the fixture stores graph/matrix hashes so a
generator drift is caught too).

    python tests/golden/make_golden.py            # writes tests/golden/*.npz
"""

from __future__ import annotations

import hashlib
import os
import signal
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import latbeam  # noqa: E402
from latbeam import decoder as D  # noqa: E402
from latbeam import lattice as LT  # noqa: E402
from latbeam import synthetic as RS  # noqa: E402

latbeam.use_numba(False)


def graph_hash(w) -> str:
    h = hashlib.sha256()
    for k in ("arc_offsets", "arc_src", "arc_dst", "arc_ilabel", "arc_olabel", "arc_weight",
              "final_cost_array"):
        h.update(np.ascontiguousarray(getattr(w, k)).tobytes())
    h.update(str(w.start_state).encode())
    return h.hexdigest()


def arr_hash(*arrs) -> str:
    h = hashlib.sha256()
    for a in arrs:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


class Timeout(Exception):
    pass


def _alarm(*_):
    raise Timeout()


def record(res):
    """Flatten a reference DecodeResult."""
    out = {"words": np.asarray(res.words, dtype=np.int64),
           "align": np.asarray(res.alignment, dtype=np.int64).reshape(-1, 2),
           "total_cost": np.float64(res.total_cost), "partial": np.int64(res.partial)}
    if res.frame_packs is not None:
        out["fp_off"] = np.cumsum([0] + [len(s) for s, _ in res.frame_packs]).astype(np.int64)
        out["fp_states"] = np.concatenate([s for s, _ in res.frame_packs]).astype(np.int64)
        out["fp_packs"] = np.concatenate([p for _, p in res.frame_packs]).astype(np.uint64)
    fl = res.lattice
    if fl is not None:
        out.update({"fl_num_nodes": np.int64(fl.num_nodes), "fl_start": np.int64(fl.start),
                    "fl_final_ids": fl.final_ids, "fl_final_costs": fl.final_costs,
                    "fl_from": fl.from_, "fl_to": fl.to, "fl_il": fl.ilabel, "fl_ol": fl.olabel,
                    "fl_g": fl.graph_cost, "fl_ac": fl.acoustic_cost,
                    "fl_node_frame": fl.node_frame, "fl_node_idx": fl.node_idx})
        # engine extras of live+pruned arcs, keyed by (block, arc id)
        lat = res.work_lattice
        keys, ext, st = [], [], []
        for b in range(len(lat.frames)):
            blk = lat.block_arrays(b)
            sel = blk["status"] != LT.STATUS_VOID
            keys.append(np.stack([np.full(sel.sum(), b), blk["arc_id"][sel]], 1))
            ext.append(blk["extra"][sel])
            st.append(blk["status"][sel])
        out["wl_keys"] = np.concatenate(keys).astype(np.int64).reshape(-1, 2)
        out["wl_extra"] = np.concatenate(ext).astype(np.float64)
        out["wl_status"] = np.concatenate(st).astype(np.int64)
    return out


def run_case(wfst, matrix, cfg, timeout=60):
    signal.signal(signal.SIGALRM, _alarm)
    signal.alarm(timeout)
    try:
        res = latbeam.decode_utterance(wfst, matrix, cfg, collect_frame_packs=True)
        return {"status": "ok", **record(res)}
    except latbeam.LatbeamError as exc:
        return {"status": type(exc).__name__, "msg": str(exc),
                "bound": getattr(exc, "bound", "")}
    except Timeout:
        return {"status": "timeout"}
    finally:
        signal.alarm(0)


def save(name, cases):
    flat = {}
    for i, c in enumerate(cases):
        for k, v in c.items():
            flat[f"{i}/{k}"] = np.asarray(v)
    flat["n"] = np.int64(len(cases))
    np.savez_compressed(os.path.join(HERE, name), **flat)
    print(f"{name}: {len(cases)} cases, {os.path.getsize(os.path.join(HERE, name)) / 1e3:.0f} kB")


def corpus_random():
    """Seeded random_task corpora from the reference's acceptance seed bases."""
    rng = np.random.default_rng(20260819)
    cases = []
    specs = []
    for seed in range(0, 120):                    # C1 base
        specs.append(dict(seed=seed, beam=float(rng.uniform(4.0, 14.0)), lattice_beam=4.0))
    for seed in range(2_000_000, 2_000_060):      # C3 base (prune_interval 4)
        specs.append(dict(seed=seed, beam=float(rng.uniform(5.0, 10.0)),
                          lattice_beam=float(rng.uniform(0.5, 6.0)), prune_interval=4))
    for seed in range(7_000_000, 7_000_060):      # eps cycles + negative costs
        specs.append(dict(seed=seed, beam=float(rng.uniform(3.0, 12.0)),
                          lattice_beam=float(rng.uniform(0.5, 6.0)), cycles=seed % 2 == 1,
                          negative=seed % 3 == 0, scale=1.0 if seed % 4 else 0.7))
    for seed in range(9_000_000, 9_000_030):      # bigger graphs, longer utterances
        specs.append(dict(seed=seed, beam=float(rng.uniform(5.0, 9.0)), lattice_beam=3.0,
                          max_states=200, max_arcs=900, max_frames=60, labels=20))
    for sp in specs:
        w, m = RS.random_task(sp["seed"], max_states=sp.get("max_states", 50),
                              max_arcs=sp.get("max_arcs", 200), num_labels=sp.get("labels", 8),
                              max_frames=sp.get("max_frames", 20),
                              allow_eps_cycles=sp.get("cycles", False),
                              allow_negative=sp.get("negative", False))
        cfg = latbeam.DecodeConfig(beam=sp["beam"], lattice_beam=sp["lattice_beam"],
                                   acoustic_scale=sp.get("scale", 1.0),
                                   prune_interval=sp.get("prune_interval", 25),
                                   max_lattice_arcs=10_000_000)
        r = run_case(w, m, cfg)
        r.update(seed=sp["seed"], beam=sp["beam"], lattice_beam=sp["lattice_beam"],
                 scale=sp.get("scale", 1.0), max_states=sp.get("max_states", 50),
                 max_arcs=sp.get("max_arcs", 200), labels=sp.get("labels", 8),
                 max_frames=sp.get("max_frames", 20), cycles=int(sp.get("cycles", False)),
                 negative=int(sp.get("negative", False)), prune_interval=sp.get("prune_interval", 25),
                 graph_hash=graph_hash(w), matrix_hash=arr_hash(m.costs))
        cases.append(r)
    return cases


def max_active_decode(wfst, matrix, beam, max_active, lattice_beam=8.0):
    """The reference frame loop (decoder.py:463-611) driven through latbeam's own
    internals, with the max-active cutoff of DESIGN.md §3 inserted after the
    emitting pass.  No lattice (1-best + frame packs)."""
    nb = 256
    beam_delta = 0.5           # Kaldi's adaptive-beam delta
    beam_eff = beam
    cfg = latbeam.DecodeConfig(beam=beam, num_workers=1, max_lattice_arcs=2_000_000)
    ws = D._Workspace(wfst)
    store = LT.ShardedArcStore(cfg.max_lattice_arcs, 1)
    lat = LT.Lattice(wfst, store)
    packs = []
    ws.reset_frame()
    ws.state_pack[wfst.start_state] = latbeam.packing.pack(0.0, 0)
    cutoff = beam
    D._eps_fixpoint(ws, wfst, store, cutoff, 0, np.array([wfst.start_state], dtype=np.int32),
                    np.array([0.0]), False)
    toks = D._aggregate(ws, wfst, cutoff, 0, wfst.start_state, cfg.max_tokens_per_frame)
    lat.append_frame(toks)
    packs.append((toks.states.copy(), ws.state_pack[toks.states].copy()))
    for t in range(1, matrix.num_frames + 1):
        acrow = matrix.costs[t - 1] * 1.0
        ws.reset_frame()
        best = D._emit(ws, wfst, toks, acrow, beam, store, cfg, None, t, False)
        store.counts[:] = 0                      # staging not needed for 1-best
        cutoff = best + beam_eff
        ss, sc, _ = D._winners(ws, cutoff, t)
        tightened = False
        if max_active and len(ss) > max_active:
            width = beam / nb
            q = (sc - best) / width
            b = np.where(q >= nb, nb - 1, q.astype(np.int64))
            cum = np.cumsum(np.bincount(b, minlength=nb))
            bstar = int(np.argmax(cum > max_active))
            h = best + float(max(bstar, 1)) * width
            if h < cutoff:
                tightened = True
                cutoff = h
                keep = sc <= cutoff
                ss, sc = ss[keep], sc[keep]
        beam_eff = min(beam, (cutoff - best) + beam_delta) if tightened else beam
        D._eps_fixpoint(ws, wfst, store, cutoff, t, ss, sc, False)
        store.counts[:] = 0
        toks = D._aggregate(ws, wfst, cutoff, t, None, cfg.max_tokens_per_frame)
        lat.append_frame(toks)
        packs.append((toks.states.copy(), ws.state_pack[toks.states].copy()))
    finals = wfst.final_cost_array[toks.states]
    totals = toks.costs + finals
    partial = not bool(np.any(np.isfinite(totals)))
    bi = int(np.argmin(toks.costs if partial else totals))
    total = float((toks.costs if partial else totals)[bi])
    words, align = D._backtrace(lat, wfst, bi)

    class R:
        pass
    r = R()
    r.words, r.alignment, r.total_cost, r.partial = words, align, total, partial
    r.frame_packs, r.lattice = packs, None
    return r


def corpus_max_active():
    cases = []
    for k, (S, deg, L, T, beam, ma) in enumerate([(2000, 5, 100, 30, 10.0, 300),
                                                  (3000, 4, 60, 25, 12.0, 500),
                                                  (1500, 6, 40, 30, 9.0, 150)]):
        w = RS.uniform_bench_graph(k, num_states=S, arcs_per_state=deg, num_labels=L)
        m = RS.bench_matrix(500 + k, num_frames=T, num_labels=L)
        r = record(max_active_decode(w, m, beam, ma))
        r.update(status="ok", kind="uniform", seed=k, S=S, deg=deg, L=L, T=T, beam=beam,
                 max_active=ma, graph_hash=graph_hash(w), matrix_hash=arr_hash(m.costs))
        cases.append(r)
    # epsilon-bearing graphs (reference random_wfst at a larger size), varied beams / caps
    prm = np.random.default_rng(4242)
    for k in range(21):
        rng = np.random.default_rng(800 + k)
        w = RS.random_wfst(rng, max_states=400, max_arcs=2400, num_labels=30)
        m = RS.random_matrix(rng, 30, max_frames=25)
        beam = 9.0 if k < 3 else float(np.round(prm.uniform(6.0, 13.0), 3))
        ma = 60 if k < 3 else int(prm.integers(15, 150))
        try:
            r = record(max_active_decode(w, m, beam, ma))
        except latbeam.LatbeamError:
            continue
        r.update(status="ok", kind="random_wfst", seed=800 + k, beam=beam, max_active=ma,
                 graph_hash=graph_hash(w), matrix_hash=arr_hash(m.costs))
        cases.append(r)
    # HCLG-shaped graphs (paper_1804_03243_b200.synthetic.hclg_graph, the C2-C5
    # generator at small size) through the reference frame loop
    sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
    from paper_1804_03243_b200 import synthetic as OS
    for k in range(16):
        S = int(prm.integers(8_000, 30_000))
        pool = int(prm.integers(300, 1200))
        ma = int(prm.integers(100, 900))
        beam = float(np.round(prm.uniform(10.0, 14.0), 3))
        T = int(prm.integers(12, 30))
        ow = OS.hclg_graph(k, num_states=S, pool_size=pool, num_pdfs=80)
        om = OS.hclg_matrix(900 + k, num_frames=T, num_pdfs=80)
        w = latbeam.Wfst(ow.num_states, ow.start_state, np.array(ow.arc_offsets), np.array(ow.arc_src),
                         np.array(ow.arc_dst), np.array(ow.arc_ilabel), np.array(ow.arc_olabel),
                         np.array(ow.arc_weight), dict(ow.final_costs))
        m = latbeam.CostMatrix(np.array(om.costs))
        try:
            r = record(max_active_decode(w, m, beam, ma))
        except latbeam.LatbeamError:
            continue
        r.update(status="ok", kind="hclg", seed=k, S=S, pool=pool, T=T, beam=beam, max_active=ma,
                 graph_hash=graph_hash(ow), matrix_hash=arr_hash(om.costs))
        cases.append(r)
    return cases


def corpus_c1(n_utts=2):
    """Config C1 at full size: uniform_bench_graph(0,10000,5,500),
    bench_matrix(100+i, 300, 500), beam 13, lattice_beam 8.  Hashes + counts only."""
    w = RS.uniform_bench_graph(0, num_states=10_000, arcs_per_state=5, num_labels=500)
    cases = []
    for i in range(n_utts):
        m = RS.bench_matrix(100 + i, num_frames=300, num_labels=500)
        cfg = latbeam.DecodeConfig(beam=13.0, lattice_beam=8.0, max_lattice_arcs=20_000_000)
        t0 = time.time()
        res = latbeam.decode_utterance(w, m, cfg, collect_frame_packs=True)
        dt = time.time() - t0
        fl = res.lattice
        fp_states = np.concatenate([s for s, _ in res.frame_packs]).astype(np.int64)
        fp_packs = np.concatenate([p for _, p in res.frame_packs]).astype(np.uint64)
        fp_off = np.cumsum([0] + [len(s) for s, _ in res.frame_packs]).astype(np.int64)
        cases.append(dict(status="ok", utt=i, words=np.asarray(res.words, dtype=np.int64),
                          align=np.asarray(res.alignment, dtype=np.int64).reshape(-1, 2),
                          total_cost=np.float64(res.total_cost), partial=np.int64(res.partial),
                          fp_off=fp_off, fp_hash=arr_hash(fp_states, fp_packs),
                          fl_num_nodes=np.int64(fl.num_nodes), fl_num_arcs=np.int64(fl.num_arcs),
                          fl_hash=arr_hash(fl.from_, fl.to, fl.ilabel, fl.olabel, fl.graph_cost,
                                           fl.acoustic_cost, fl.final_ids, fl.final_costs),
                          ref_seconds=dt, graph_hash=graph_hash(w), matrix_hash=arr_hash(m.costs)))
        print(f"C1 utt {i}: {dt:.1f}s, {fl.num_arcs} arcs, cost {res.total_cost}")
    return cases


def corpus_text():
    """write_lattice_text (lattice.py:605-614) of the reference's own FinalLattice,
    pinned by sha256 + length: random tasks and config C1's first utterance cut
    to 40 frames (~50k-arc text)."""
    import hashlib as _h
    cases = []
    for seed in range(3_000_000, 3_000_040):
        w, m = RS.random_task(seed)
        cfg = latbeam.DecodeConfig(beam=9.0, lattice_beam=4.0)
        try:
            res = latbeam.decode_utterance(w, m, cfg)
        except latbeam.LatbeamError:
            continue
        txt = latbeam.write_lattice_text(res.lattice).encode()
        cases.append(dict(kind="random", seed=seed, beam=9.0, lattice_beam=4.0, sha=_h.sha256(txt).hexdigest(),
                          length=len(txt), graph_hash=graph_hash(w), matrix_hash=arr_hash(m.costs)))
    w = RS.uniform_bench_graph(0, num_states=10_000, arcs_per_state=5, num_labels=500)
    m = latbeam.CostMatrix(RS.bench_matrix(100, num_frames=300, num_labels=500).costs[:40].copy())
    res = latbeam.decode_utterance(w, m, latbeam.DecodeConfig(beam=13.0, lattice_beam=8.0,
                                                              max_lattice_arcs=20_000_000))
    txt = latbeam.write_lattice_text(res.lattice).encode()
    cases.append(dict(kind="c1_40", seed=0, beam=13.0, lattice_beam=8.0, sha=_h.sha256(txt).hexdigest(),
                      length=len(txt), graph_hash=graph_hash(w), matrix_hash=arr_hash(m.costs)))
    print(f"text corpus: {len(cases)} lattices, C1/40 text {len(txt)} bytes")
    return cases


if __name__ == "__main__":
    which = sys.argv[1:] or ["random", "max_active", "c1"]
    if "random" in which:
        save("random_tasks.npz", corpus_random())
    if "max_active" in which:
        save("max_active.npz", corpus_max_active())
    if "c1" in which:
        save("c1.npz", corpus_c1())
    if "text" in which:
        save("lattice_text.npz", corpus_text())
