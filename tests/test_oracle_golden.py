"""Pin the CPU oracle (oracle/) to the reference implementation's own outputs.

The fixtures under tests/golden/ were produced by tests/golden/make_golden.py,
which runs the reference package `latbeam` (/root/reference, numpy engine) on
seeded inputs.  Inputs are regenerated here by this package's restated
generators; their hashes must match the reference generators' (so the seeds
name the same graphs), and the oracle must reproduce the reference bit-exactly:
words, alignment, total cost, partial flag, every frame's (state, packed word)
map and the finalized lattice arrays; work-lattice extras within 1e-9.
"""

import hashlib
import os

import numpy as np
import pytest

from paper_1804_03243_b200 import synthetic

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
ERRNAMES = {1: "DecodeFailure", 2: "UsageError", 3: "CapacityError", 4: "InternalInvariantError"}


def load(name):
    z = np.load(os.path.join(GOLD, name), allow_pickle=False)
    n = int(z["n"])
    cases = [{} for _ in range(n)]
    for k in z.files:
        if k == "n":
            continue
        i, key = k.split("/", 1)
        cases[int(i)][key] = z[k]
    return cases


def graph_hash(w):
    h = hashlib.sha256()
    for k in ("arc_offsets", "arc_src", "arc_dst", "arc_ilabel", "arc_olabel", "arc_weight",
              "final_cost_array"):
        h.update(np.ascontiguousarray(getattr(w, k)).tobytes())
    h.update(str(w.start_state).encode())
    return h.hexdigest()


def arr_hash(*arrs):
    h = hashlib.sha256()
    for a in arrs:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def check_case(c, res):
    st = str(c["status"])
    if st == "timeout":
        pytest.skip("reference timed out on this case")
    if st != "ok":
        assert not res.ok and ERRNAMES[res.status] == st, (res.status, res.message, st)
        return
    assert res.ok, res.message
    assert res.words == c["words"].tolist()
    assert res.alignment == [tuple(x) for x in c["align"].tolist()]
    assert res.total_cost == float(c["total_cost"])
    assert res.partial == bool(c["partial"])
    states = np.concatenate([f[0] for f in res.frames]).astype(np.int64)
    packs = np.concatenate([f[4] for f in res.frames])
    off = np.cumsum([0] + [len(f[0]) for f in res.frames])
    assert np.array_equal(off, c["fp_off"])
    assert np.array_equal(states, c["fp_states"])
    assert np.array_equal(packs, c["fp_packs"])
    if "fl_from" in c:
        fl = res.final
        assert fl["num_nodes"] == int(c["fl_num_nodes"]) and fl["start"] == int(c["fl_start"])
        for mine, theirs in (("final_ids", "fl_final_ids"), ("final_costs", "fl_final_costs"),
                             ("from_", "fl_from"), ("to", "fl_to"), ("ilabel", "fl_il"),
                             ("olabel", "fl_ol"), ("graph_cost", "fl_g"), ("acoustic_cost", "fl_ac"),
                             ("node_frame", "fl_node_frame"), ("node_idx", "fl_node_idx")):
            assert np.array_equal(fl[mine], c[theirs]), mine
        # engine extras of every non-void arc, by (block, arc id)
        keys, ext = [], []
        for b, blk in enumerate(res.blocks):
            keys.append(np.stack([np.full(len(blk[0]), b), blk[0]], 1))
            ext.append(blk[4])
        keys = np.concatenate(keys)
        ext = np.concatenate(ext)
        pruned = np.concatenate([blk[5] for blk in res.blocks])
        ref_keys, ref_ext, ref_st = c["wl_keys"], c["wl_extra"], c["wl_status"]
        o1 = np.lexsort((keys[:, 1], keys[:, 0]))
        o2 = np.lexsort((ref_keys[:, 1], ref_keys[:, 0]))
        assert np.array_equal(keys[o1], ref_keys[o2])
        # the reference prunes every prune_interval frames and keeps a pruned
        # arc's mid-decode extra (a lower bound); the oracle prunes once from
        # the final terminus, so only LIVE arcs carry comparable extras
        # (the reference's own C3 rule, test_acceptance.py:146-150)
        assert np.array_equal(pruned[o1], ref_st[o2] == 1)
        live = ref_st[o2] == 0
        e1, e2 = ext[o1][live], ref_ext[o2][live]
        assert np.all(np.isfinite(e1) == np.isfinite(e2))
        if len(e2):
            assert np.max(np.abs(e1 - e2)) <= 1e-9


CASES = load("random_tasks.npz")


@pytest.mark.parametrize("idx", range(len(CASES)))
def test_random_task_golden(oracle_mod, idx):
    c = CASES[idx]
    w, m = synthetic.random_task(int(c["seed"]), max_states=int(c["max_states"]),
                                 max_arcs=int(c["max_arcs"]), num_labels=int(c["labels"]),
                                 max_frames=int(c["max_frames"]), allow_eps_cycles=bool(c["cycles"]),
                                 allow_negative=bool(c["negative"]))
    assert graph_hash(w) == str(c["graph_hash"]), "generator restatement drifted from reference"
    assert arr_hash(m.costs) == str(c["matrix_hash"])
    res = oracle_mod.decode(w, m, float(c["beam"]), lattice_beam=float(c["lattice_beam"]),
                            acoustic_scale=float(c["scale"]), max_lattice_arcs=10_000_000)
    check_case(c, res)


def test_golden_corpus_is_substantive():
    kinds = [str(c["status"]) for c in CASES]
    assert kinds.count("ok") >= 200
    assert sum(1 for c in CASES if str(c["status"]) == "ok" and int(c["partial"])) >= 1
    assert sum(1 for c in CASES if int(c.get("cycles", 0))) >= 20


MA_CASES = load("max_active.npz")


def test_max_active_corpus_is_substantive():
    kinds = [str(c["kind"]) for c in MA_CASES]
    assert len(MA_CASES) >= 40 and kinds.count("hclg") >= 12 and kinds.count("random_wfst") >= 20


@pytest.mark.parametrize("idx", range(len(MA_CASES)))
def test_max_active_extension_golden(oracle_mod, idx):
    """Max-active extension vs the reference frame loop with the DESIGN.md §3 cutoff."""
    c = MA_CASES[idx]
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
    res = oracle_mod.decode(w, m, float(c["beam"]), max_active=int(c["max_active"]),
                            want_lattice=False)
    check_case(c, res)
    if str(c["kind"]) == "uniform":   # the cap must bind for the fixture to mean anything
        assert max(len(f[0]) for f in res.frames) < 0.5 * w.num_states


@pytest.mark.parametrize("utt", [0, 1])
def test_config1_full_utterance_golden(oracle_mod, utt):
    """Config C1 at full size (10k states, 300 frames, beam 13, lattice beam 8)."""
    c = load("c1.npz")[utt]
    w = synthetic.config_graph("C1")
    m = synthetic.config_matrix("C1", utt)
    assert graph_hash(w) == str(c["graph_hash"]) and arr_hash(m.costs) == str(c["matrix_hash"])
    res = oracle_mod.decode(w, m, 13.0, lattice_beam=8.0)
    assert res.ok
    assert res.words == c["words"].tolist() and res.total_cost == float(c["total_cost"])
    assert res.alignment == [tuple(x) for x in c["align"].tolist()]
    states = np.concatenate([f[0] for f in res.frames]).astype(np.int64)
    packs = np.concatenate([f[4] for f in res.frames])
    assert arr_hash(states, packs) == str(c["fp_hash"])
    fl = res.final
    assert fl["num_nodes"] == int(c["fl_num_nodes"]) and len(fl["from_"]) == int(c["fl_num_arcs"])
    assert arr_hash(fl["from_"], fl["to"], fl["ilabel"], fl["olabel"], fl["graph_cost"],
                    fl["acoustic_cost"], fl["final_ids"], fl["final_costs"]) == str(c["fl_hash"])


TEXT_CASES = load("lattice_text.npz")


def _text_inputs(c):
    if str(c["kind"]) == "random":
        w, m = synthetic.random_task(int(c["seed"]))
    else:
        w = synthetic.config_graph("C1")
        m = synthetic.CostMatrix(synthetic.config_matrix("C1", 0).costs[:40].copy())
    assert graph_hash(w) == str(c["graph_hash"]) and arr_hash(m.costs) == str(c["matrix_hash"])
    return w, m


@pytest.mark.parametrize("idx", range(len(TEXT_CASES)))
def test_lattice_text_golden(oracle_mod, idx):
    """The reference's write_lattice_text of its own lattice (sha256 + length,
    tests/golden/make_golden.py corpus_text) equals the native text writer
    (lb_lattice_text, host-only) over the oracle's FinalLattice: pins the
    finalised arrays and the Python-repr float formatting at once, up to a
    ~140k-arc C1 lattice."""
    import hashlib

    import paper_1804_03243_b200 as lb
    c = TEXT_CASES[idx]
    w, m = _text_inputs(c)
    ref = oracle_mod.decode(w, m, float(c["beam"]), lattice_beam=float(c["lattice_beam"]),
                            max_lattice_arcs=20_000_000)
    assert ref.ok
    f = ref.final
    fl = lb.FinalLattice(f["num_nodes"], f["start"], f["final_ids"], f["final_costs"], f["from_"], f["to"],
                         f["ilabel"], f["olabel"], f["graph_cost"], f["acoustic_cost"])
    txt = lb.write_lattice_text(fl).encode()
    assert len(txt) == int(c["length"])
    assert hashlib.sha256(txt).hexdigest() == str(c["sha"])
