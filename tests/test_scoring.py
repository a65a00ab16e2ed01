"""Lattice scoring (scoring.py of `latbeam`): the CPU restatement pinned to the
reference's golden vectors, the host functions, and the GPU oracle-WER kernel
(csrc/lb_scoring.cuh) against both."""

from __future__ import annotations

import os

import numpy as np
import pytest

import paper_1804_03243_b200 as lb
from oracle import scoring_oracle as SO
from paper_1804_03243_b200.lattice import FinalLattice

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = np.load(os.path.join(HERE, "golden", "scoring.npz"))
N = int(GOLD["n"])


def case(i):
    g = {k: GOLD[f"{i}/{k}"] for k in ("num_nodes", "start", "final_ids", "from_", "to", "ilabel", "olabel",
                                       "node_frame", "ref", "hyp", "oracle_wer", "wer", "density")}
    m = len(g["from_"])
    fl = FinalLattice(int(g["num_nodes"]), int(g["start"]), g["final_ids"], np.zeros(len(g["final_ids"])),
                      g["from_"], g["to"], g["ilabel"], g["olabel"], np.zeros(m), np.zeros(m),
                      node_frame=g["node_frame"], num_frames=int(g["node_frame"].max()))
    return g, fl


def test_golden_set_is_meaningful():
    ows = [int(GOLD[f"{i}/oracle_wer"]) for i in range(N)]
    assert N >= 60
    assert len(set(ows)) > 5 and 0 in ows
    assert max(len(GOLD[f"{i}/from_"]) for i in range(N)) > 500


@pytest.mark.parametrize("i", range(N))
def test_oracle_restatement_matches_reference_golden(i):
    g, fl = case(i)
    ow = SO.oracle_wer(fl.num_nodes, fl.start, fl.final_ids, fl.from_, fl.to, fl.olabel, list(g["ref"]))
    assert (ow if ow is not None else -1) == int(g["oracle_wer"])
    s, ins, d = SO.wer(list(g["hyp"]), list(g["ref"]))
    assert [s, ins, d] == g["wer"].tolist()


@pytest.mark.parametrize("i", range(N))
def test_host_wer_and_density_match_reference_golden(i):
    g, fl = case(i)
    r = lb.wer([int(x) for x in g["hyp"]], [int(x) for x in g["ref"]])
    assert [r.substitutions, r.insertions, r.deletions] == g["wer"].tolist()
    assert lb.wer_percent(list(g["hyp"]), list(g["ref"])) == 100.0 * r.errors / len(g["ref"])
    assert lb.lattice_density(fl) == float(g["density"])


def test_wer_tie_order_and_errors():
    assert lb.wer([1, 2, 3], [1, 2, 3]) == lb.WerResult(0, 0, 0)
    assert lb.wer([], [1, 2]) == lb.WerResult(0, 0, 2)
    assert lb.wer([1, 2], [3]) == lb.WerResult(1, 1, 0)
    rng = np.random.default_rng(7)
    for _ in range(200):
        h = rng.integers(1, 5, rng.integers(0, 9)).tolist()
        r = rng.integers(1, 5, rng.integers(1, 9)).tolist()
        assert tuple(lb.wer(h, r).__dict__.values()) == SO.wer(h, r)
    with pytest.raises(lb.UsageError):
        lb.wer([1], [])


def test_density_errors():
    _, fl = case(0)
    with pytest.raises(lb.UsageError):
        lb.lattice_density(fl, num_frames=0)
    assert lb.lattice_density(fl, num_frames=2) == fl.num_arcs / 2.0


def test_usage_errors_before_device():
    _, fl = case(0)
    with pytest.raises(lb.UsageError):
        lb.oracle_wer(fl, [])
    with pytest.raises(lb.UsageError):
        lb.oracle_wer_batch([fl], [[1], [2]])
    assert lb.oracle_wer_batch([], []) == []


# ---------------------------------------------------------------- GPU kernel

def _oracle(fl, ref):
    ow = SO.oracle_wer(fl.num_nodes, fl.start, fl.final_ids, fl.from_, fl.to, fl.olabel, ref)
    return -1 if ow is None else ow


def _gpu_or_minus1(fl, ref):
    try:
        return lb.oracle_wer(fl, ref)
    except lb.UsageError as e:
        assert "no complete path" in str(e)
        return -1


@pytest.mark.gpu
def test_gpu_oracle_wer_batch_matches_reference_golden():
    cases = [case(i) for i in range(N)]
    ok = [(g, fl) for g, fl in cases if int(g["oracle_wer"]) >= 0]
    got = lb.oracle_wer_batch([fl for _, fl in ok], [[int(x) for x in g["ref"]] for g, _ in ok])
    assert got == [int(g["oracle_wer"]) for g, _ in ok]
    for g, fl in cases:
        assert _gpu_or_minus1(fl, [int(x) for x in g["ref"]]) == int(g["oracle_wer"])


@pytest.mark.gpu
def test_gpu_oracle_wer_unframed_and_shuffled_lattices():
    """Node ids out of frame order / arcs unsorted / no node_frame: the kernel's
    whole-lattice fixpoint path must give the reference's numbers too."""
    rng = np.random.default_rng(3)
    for i in range(N):
        g, fl = case(i)
        perm = rng.permutation(fl.num_nodes)
        ap = rng.permutation(fl.num_arcs)
        sh = FinalLattice(fl.num_nodes, int(perm[fl.start]), perm[fl.final_ids], fl.final_costs,
                          perm[fl.from_][ap], perm[fl.to][ap], fl.ilabel[ap], fl.olabel[ap], fl.graph_cost,
                          fl.acoustic_cost, node_frame=None)
        assert _gpu_or_minus1(sh, [int(x) for x in g["ref"]]) == int(g["oracle_wer"])


@pytest.mark.gpu
def test_gpu_oracle_wer_on_decoded_lattices():
    """GPU-decoded lattices (config-C1-like graph), long references, scored on the
    GPU in one batch and by the CPU restatement."""
    from paper_1804_03243_b200 import synthetic
    g = synthetic.hclg_graph(11, num_states=20000, num_pdfs=80, pool_size=2000, num_words=300)
    mats = [synthetic.hclg_matrix(500 + i, num_frames=60, num_pdfs=80) for i in range(6)]
    res = lb.decode_batch(g, mats, lb.DecodeConfig(beam=11.0, lattice_beam=6.0, max_active=3000))
    rng = np.random.default_rng(5)
    lats, refs = [], []
    for r in res:
        words = r.words or [1]
        ref = [int(words[rng.integers(len(words))]) if rng.random() < 0.8 else int(rng.integers(1, 300))
               for _ in range(max(1, len(words) + int(rng.integers(-3, 4))))]
        lats.append(r.lattice)
        refs.append(ref)
    assert max(fl.num_arcs for fl in lats) > 1000
    got = lb.oracle_wer_batch(lats, refs)
    assert got == [_oracle(fl, ref) for fl, ref in zip(lats, refs)]
    # the 1-best path is in the lattice, so the oracle can only do better
    for r, ref, ow in zip(res, refs, got):
        assert ow <= lb.wer(r.words, ref).errors
