"""Parity at BASELINE.json's full config sizes (C1-C5), device vs the CPU oracle.

Every config runs its real graph (SURVEY.md §8(d) generators, full size) and
real-length utterances:

* C1  uniform 10k x 5, 500 pdfs, beam 13, lattice beam 8: all 20 utterances x
      300 frames 1-best bit-exact (cost + work counters), two of them with
      per-frame packs and the full lattice.
* C2  HCLG 5M states, beam 13, max-active 7000, 1-best: one 300-frame utterance,
      per-frame (state, pack) maps bit-exact.
* C3  C2 + lattice beam 8: one 300-frame utterance, lattice arc sets / extras.
* C4  C2 graph, sequence-parallel batch: 64 utterances in one launch (64 lanes),
      every total cost and work counter bit-exact vs the threaded oracle.
* C4r the C4 graph with a ragged 192-utterance job on 64 refilling lanes.
* C5  HCLG 15M states / ~50M arcs with 1000 epsilon hubs (in-degree ~8.5k) and
      depth-8 epsilon chains, beam 16, max-active 20000: one 300-frame utterance
      bit-exact.
"""

from __future__ import annotations

import time

import numpy as np
import pytest

import paper_1804_03243_b200 as lb
from paper_1804_03243_b200 import synthetic

from parity_helpers import check_pair, decode_both

pytestmark = pytest.mark.gpu

_GRAPHS: dict = {}


@pytest.fixture(scope="module", autouse=True)
def _release_graphs():
    """Drop the full-size graphs (and their device replicas + lane workspaces,
    tens of GB at C4) before the next test module runs."""
    yield
    import gc
    _GRAPHS.clear()
    gc.collect()


def graph(name):
    key = "C2" if name in ("C2", "C3", "C4") else name
    if key not in _GRAPHS:
        _GRAPHS[key] = synthetic.config_graph(key)
    return _GRAPHS[key]


def _counters(r):
    """Work counters that are a pure function of the token lists: tokens expanded,
    arcs scanned, tokens kept (the device skips hopeless atomics, so its candidate
    and epsilon-offer counts are legitimately lower than the oracle's)."""
    c = r.counters
    return [c["n_tokens"], c["n_scan"], c["n_next"]]


def test_c1_all_utterances(oracle_mod):
    w = graph("C1")
    d = synthetic.CONFIGS["C1"]["decode"]
    mats = [synthetic.config_matrix("C1", u) for u in range(20)]
    tc, st, cnt = oracle_mod.decode_batch_mt(w, mats, d["beam"])
    res = lb.decode_batch(w, mats, lb.DecodeConfig(beam=d["beam"]), want_lattice=False)
    assert all(st == 0)
    assert [r.total_cost for r in res] == tc.tolist()
    for r, c in zip(res, cnt):
        assert _counters(r) == [c[0], c[1], c[6]]
    for u in range(2):
        got, ref = decode_both(w, mats[u], oracle_mod, d["beam"], d["lattice_beam"])
        check_pair(got, ref, d["lattice_beam"])


@pytest.mark.parametrize("name,want_lattice", [("C2", False), ("C3", True)])
def test_c2_c3_full_utterance(oracle_mod, name, want_lattice):
    w = graph(name)
    d = synthetic.CONFIGS[name]["decode"]
    m = synthetic.config_matrix(name, 0)
    got, ref = decode_both(w, m, oracle_mod, d["beam"], d["lattice_beam"],
                           max_active=d["max_active"], want_lattice=want_lattice)
    check_pair(got, ref, d["lattice_beam"], want_lattice=want_lattice)
    # max-active binds on this graph: the cap is reached on most frames
    sizes = np.asarray([len(s) for s, _ in got.frame_packs[1:]])
    assert np.median(sizes) >= 0.9 * d["max_active"], np.median(sizes)


def test_c3_lattice_oracle_wer_on_gpu():
    """Full-size C3 lattice (HCLG graph, epsilon arcs, lattice beam 8): GPU oracle
    WER vs the CPU restatement of scoring.py:66-114, against a reference made
    from the 1-best words with seeded edits."""
    from oracle import scoring_oracle as SO
    w = graph("C3")
    d = synthetic.CONFIGS["C3"]["decode"]
    r = lb.decode_utterance(w, synthetic.config_matrix("C3", 0),
                            lb.DecodeConfig(beam=d["beam"], lattice_beam=d["lattice_beam"],
                                            max_active=d["max_active"], max_lattice_arcs=50_000_000))
    fl = r.lattice
    assert fl.num_arcs > 10000
    rng = np.random.default_rng(9)
    ref = [x if rng.random() < 0.7 else int(rng.integers(1, 1000)) for x in r.words[:12]] or [1]
    t0 = time.perf_counter()
    got = lb.oracle_wer(fl, ref)
    print(f"C3 lattice {fl.num_nodes} nodes {fl.num_arcs} arcs: gpu oracle_wer {time.perf_counter() - t0:.3f}s")
    t0 = time.perf_counter()
    want = SO.oracle_wer(fl.num_nodes, fl.start, fl.final_ids, fl.from_, fl.to, fl.olabel, ref)
    print(f"cpu restatement {time.perf_counter() - t0:.3f}s")
    assert got == want
    assert got <= lb.wer(r.words, ref).errors


def test_c4_batch_of_64_lanes(oracle_mod):
    w = graph("C4")
    d = synthetic.CONFIGS["C4"]["decode"]
    mats = [synthetic.config_matrix("C4", u) for u in range(64)]
    tc, st, cnt = oracle_mod.decode_batch_mt(w, mats, d["beam"], max_active=d["max_active"])
    res = lb.decode_batch(w, mats, lb.DecodeConfig(beam=d["beam"], max_active=d["max_active"],
                                                   lanes=64), want_lattice=False)
    assert all(st == 0)
    assert [r.total_cost for r in res] == tc.tolist()
    for r, c in zip(res, cnt):
        assert _counters(r) == [c[0], c[1], c[6]]


def test_c5_stress_utterance(oracle_mod):
    w = graph("C5")
    assert w.num_arcs > 45_000_000  # ~49.9M
    d = synthetic.CONFIGS["C5"]["decode"]
    m = synthetic.config_matrix("C5", 0)
    got, ref = decode_both(w, m, oracle_mod, d["beam"], d["lattice_beam"],
                           max_active=d["max_active"], want_lattice=False)
    check_pair(got, ref, d["lattice_beam"], want_lattice=False)
    assert ref.counters["eps_scan"] > 0
    # the stress shape SURVEY.md §8(d) asks for: ~1000 epsilon "backoff" hubs of
    # in-degree ~1e4 (measured here: ~8.5k each, every hub at least 8k)
    eps = w.arc_ilabel == 0
    indeg = np.sort(np.bincount(w.arc_dst[eps], minlength=w.num_states))[-1000:]
    print(f"C5 hubs: epsilon in-degree of the top 1000 states mean {indeg.mean():.0f} min {indeg.min()}")
    assert indeg.mean() >= 8000 and indeg.min() >= 7000


def test_c4_ragged_refill_full_graph(oracle_mod):
    """C4's graph with a ragged job larger than the lane count: 192 utterances,
    T ~ U[100, 500], 64 lanes -> one refilling launch (44 two-CTA + 20 three-CTA
    lanes on one queue) fed through the streamed pinned ring; every total cost and
    work counter equals the threaded oracle, in input order."""
    w = graph("C4")
    d = synthetic.CONFIGS["C4"]["decode"]
    rng = np.random.default_rng(404)
    mats = [np.ascontiguousarray(synthetic.hclg_matrix(5000 + u, num_frames=int(rng.integers(100, 501))).costs)
            for u in range(192)]
    tc, st, cnt = oracle_mod.decode_batch_mt(w, mats, d["beam"], max_active=d["max_active"])
    res = lb.decode_batch(w, mats, lb.DecodeConfig(beam=d["beam"], max_active=d["max_active"], lanes=64),
                          want_lattice=False)
    assert all(st == 0)
    assert [r.total_cost for r in res] == tc.tolist()
    for r, c in zip(res, cnt):
        assert _counters(r) == [c[0], c[1], c[6]]


@pytest.mark.parametrize("n,mode,want_lattice", [(44, None, True), (64, "batched", False)])
def test_c1_large_batched_batches(oracle_mod, monkeypatch, n, mode, want_lattice):
    """C1's dense 10k-state graph (~48k candidates per lane-frame, no max-active) in
    the batched mode at 44 / 64 lanes: its candidate buffers hold every warp's
    partly used chunk (a round-2 sweep found 44+ lanes overflowing them)."""
    if mode:
        monkeypatch.setenv("LB_MODE", mode)
    w = graph("C1")
    d = synthetic.CONFIGS["C1"]["decode"]
    mats = [np.ascontiguousarray(synthetic.config_matrix("C1", u % 20, num_frames=60).costs) for u in range(n)]
    res = lb.decode_batch(w, mats, lb.DecodeConfig(beam=d["beam"], lattice_beam=d["lattice_beam"],
                                                   max_lattice_arcs=20_000_000), want_lattice=want_lattice)
    tc, st, _ = oracle_mod.decode_batch_mt(w, mats, d["beam"])
    assert all(st == 0)
    assert [r.total_cost for r in res] == tc.tolist()
