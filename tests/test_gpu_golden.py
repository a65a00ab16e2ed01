"""The CUDA path against the reference's OWN outputs (tests/golden/, produced by
running `latbeam` itself; see make_golden.py), not only against the oracle:
every max-active case (uniform, random epsilon graphs, HCLG-shaped graphs
through the reference frame loop with the DESIGN.md §3 cutoff) and the
random-task corpus, in both device modes.  Bit-exact words, alignment, total
cost, partial flag and every frame's (state, packed word) map."""

import numpy as np
import pytest

import paper_1804_03243_b200 as lb
from paper_1804_03243_b200 import synthetic
from test_oracle_golden import CASES, MA_CASES, arr_hash, graph_hash

pytestmark = pytest.mark.gpu
ERR = {"DecodeFailure": lb.DecodeFailure, "UsageError": lb.UsageError,
       "CapacityError": lb.CapacityError, "InternalInvariantError": lb.InternalInvariantError}


def _check(c, got):
    st = str(c["status"])
    if st == "timeout":
        return "skip"
    if st != "ok":
        assert isinstance(got, ERR[st]), (got, st)
        return "error"
    assert not isinstance(got, Exception), got
    assert got.words == c["words"].tolist()
    assert got.alignment == [tuple(x) for x in c["align"].tolist()]
    assert got.total_cost == float(c["total_cost"])
    assert got.partial == bool(c["partial"])
    states = np.concatenate([s for s, _ in got.frame_packs]).astype(np.int64)
    packs = np.concatenate([p for _, p in got.frame_packs])
    off = np.cumsum([0] + [len(s) for s, _ in got.frame_packs])
    assert np.array_equal(off, c["fp_off"])
    assert np.array_equal(states, c["fp_states"]) and np.array_equal(packs, c["fp_packs"])
    return "ok"


def _ma_inputs(c):
    if str(c["kind"]) == "uniform":
        w = synthetic.uniform_bench_graph(int(c["seed"]), num_states=int(c["S"]),
                                          arcs_per_state=int(c["deg"]), num_labels=int(c["L"]))
        m = synthetic.bench_matrix(500 + int(c["seed"]), num_frames=int(c["T"]), num_labels=int(c["L"]))
    elif str(c["kind"]) == "hclg":
        w = synthetic.hclg_graph(int(c["seed"]), num_states=int(c["S"]), pool_size=int(c["pool"]), num_pdfs=80)
        m = synthetic.hclg_matrix(900 + int(c["seed"]), num_frames=int(c["T"]), num_pdfs=80)
    else:
        rng = np.random.default_rng(int(c["seed"]))
        w = synthetic.random_wfst(rng, max_states=400, max_arcs=2400, num_labels=30)
        m = synthetic.random_matrix(rng, 30, max_frames=25)
    assert graph_hash(w) == str(c["graph_hash"]) and arr_hash(m.costs) == str(c["matrix_hash"])
    return w, m


@pytest.mark.parametrize("mode", ["batched", "lane"])
def test_max_active_golden_on_device(monkeypatch, mode):
    monkeypatch.setenv("LB_MODE", mode)
    n = 0
    for c in MA_CASES:
        w, m = _ma_inputs(c)
        cfg = lb.DecodeConfig(beam=float(c["beam"]), max_active=int(c["max_active"]))
        try:
            got = lb.decode_utterance(w, m, cfg, want_lattice=False, collect_frame_packs=True)
        except lb.LatbeamError as exc:
            got = exc
        n += _check(c, got) == "ok"
    assert n >= 40


@pytest.mark.parametrize("mode", ["batched", "lane"])
def test_random_task_golden_on_device(monkeypatch, mode):
    monkeypatch.setenv("LB_MODE", mode)
    kinds = {}
    for c in CASES[::3]:
        w, m = synthetic.random_task(int(c["seed"]), max_states=int(c["max_states"]),
                                     max_arcs=int(c["max_arcs"]), num_labels=int(c["labels"]),
                                     max_frames=int(c["max_frames"]), allow_eps_cycles=bool(c["cycles"]),
                                     allow_negative=bool(c["negative"]))
        cfg = lb.DecodeConfig(beam=float(c["beam"]), lattice_beam=float(c["lattice_beam"]),
                              acoustic_scale=float(c["scale"]))
        try:
            got = lb.decode_utterance(w, m, cfg, want_lattice=False, collect_frame_packs=True)
        except lb.LatbeamError as exc:
            got = exc
        k = _check(c, got)
        kinds[k] = kinds.get(k, 0) + 1
    assert kinds.get("ok", 0) >= 60, kinds


def test_lattice_text_golden_on_device():
    """Device-decoded lattices written as text equal the reference's own text
    (sha256), random tasks and a 40-frame C1 lattice."""
    import hashlib

    from test_oracle_golden import TEXT_CASES, _text_inputs
    for c in TEXT_CASES:
        w, m = _text_inputs(c)
        r = lb.decode_utterance(w, m, lb.DecodeConfig(beam=float(c["beam"]), lattice_beam=float(c["lattice_beam"]),
                                                      max_lattice_arcs=20_000_000))
        txt = lb.write_lattice_text(r.lattice).encode()
        assert len(txt) == int(c["length"]) and hashlib.sha256(txt).hexdigest() == str(c["sha"])
