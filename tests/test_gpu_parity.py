"""Parity of the CUDA path (liblatbeam_b200.so via the public API) with the CPU oracle.

Bit-exact: words, alignment, total_cost, partial and every frame's
(state, packed word) map.  Lattices: identical FinalLattice arrays unless an
oracle extra lies within 1e-3 of lattice_beam (the reference's C3 rule,
test_acceptance.py:151-165); live-arc extras within 1e-4 always.
"""

import math

import numpy as np
import pytest

import paper_1804_03243_b200 as lb
from paper_1804_03243_b200 import synthetic
from parity_helpers import check_pair, compare_1best, decode_both

pytestmark = pytest.mark.gpu


def test_native_library_is_the_path():
    from paper_1804_03243_b200 import _lib
    L = _lib.lib()
    assert L.lb_device_count() >= 1
    assert L.lb_version() == 1


@pytest.mark.parametrize("mode", ["batched", "lane"])
@pytest.mark.parametrize("base,cycles,negative", [(0, False, False), (1_000_000, False, True),
                                                  (7_000_000, True, False), (3_000_000, True, True)])
def test_random_corpus(oracle_mod, monkeypatch, mode, base, cycles, negative):
    """1-best + lattice on random graphs, through both device modes."""
    monkeypatch.setenv("LB_MODE", mode)
    rng = np.random.default_rng(base + 17)
    kinds = {}
    for seed in range(base, base + 60):
        w, m = synthetic.random_task(seed, allow_eps_cycles=cycles, allow_negative=negative)
        beam = float(rng.uniform(3.0, 14.0))
        lbeam = float(rng.uniform(0.0, 6.0))
        scale = 1.0 if seed % 3 else 0.75
        got, ref = decode_both(w, m, oracle_mod, beam, lbeam, scale)
        k = check_pair(got, ref, lbeam)
        kinds[k] = kinds.get(k, 0) + 1
    assert kinds.get("exact", 0) >= 20, kinds


@pytest.mark.parametrize("mode", ["batched", "lane"])
@pytest.mark.parametrize("base,cycles,negative", [(11_000_000, True, False), (12_000_000, False, True)])
def test_random_corpus_1best_modes(oracle_mod, monkeypatch, mode, base, cycles, negative):
    """1-best decodes (per-frame packs bit-exact) through both device modes: the
    frame-synchronous batched kernels and the persistent-lane kernel."""
    monkeypatch.setenv("LB_MODE", mode)
    rng = np.random.default_rng(base)
    for seed in range(base, base + 40):
        w, m = synthetic.random_task(seed, allow_eps_cycles=cycles, allow_negative=negative)
        beam = float(rng.uniform(3.0, 14.0))
        scale = 1.0 if seed % 3 else 0.75
        got, ref = decode_both(w, m, oracle_mod, beam, 4.0, scale, want_lattice=False,
                               max_active=int(rng.integers(0, 12)))
        check_pair(got, ref, 4.0, want_lattice=False)


@pytest.mark.parametrize("threads", [512, 640, 768])
def test_lane_cta_sizes(oracle_mod, monkeypatch, threads):
    """Every supported lane CTA size (kernel template variant) decodes 1-best and
    lattices bit-exactly vs the oracle, epsilon cycles and max-active included."""
    monkeypatch.setenv("LB_MODE", "lane")
    rng = np.random.default_rng(threads)
    for seed in range(13_000_000, 13_000_025):
        w, m = synthetic.random_task(seed, allow_eps_cycles=seed % 2 == 0)
        beam = float(rng.uniform(4.0, 13.0))
        got, ref = decode_both(w, m, oracle_mod, beam, 3.0, max_active=int(rng.integers(0, 10)),
                               device_kw={"threads_per_lane": threads})
        check_pair(got, ref, 3.0)


@pytest.mark.parametrize("ctas", [3, 4, 8, 16])
def test_wide_lane_clusters(oracle_mod, monkeypatch, ctas):
    """3-, 4-, 8- and 16-CTA lane clusters (picked automatically for batches of up
    to 45 utterances; 16 CTAs is a non-portable cluster size) decode 1-best and
    lattices bit-exactly vs the oracle."""
    monkeypatch.setenv("LB_MODE", "lane")
    rng = np.random.default_rng(ctas)
    for seed in range(14_000_000, 14_000_020):
        w, m = synthetic.random_task(seed, allow_eps_cycles=seed % 2 == 1)
        beam = float(rng.uniform(4.0, 13.0))
        got, ref = decode_both(w, m, oracle_mod, beam, 3.0, max_active=int(rng.integers(0, 10)),
                               device_kw={"ctas_per_lane": ctas})
        check_pair(got, ref, 3.0)


@pytest.mark.parametrize("n", [1, 3, 8, 20, 40])
def test_auto_mode_batches(oracle_mod, n):
    """The automatic mode choice (16-CTA lanes at 1 and 3, 8-CTA lanes at 8, 4-CTA
    lanes at 20, 3-CTA lanes at 40 utterances) gives the oracle's costs and work
    counters."""
    w = synthetic.hclg_graph(4, num_states=300_000, pool_size=4000, num_pdfs=500)
    mats = [synthetic.hclg_matrix(700 + i, num_frames=30 + (i % 7), num_pdfs=500) for i in range(n)]
    cfg = lb.DecodeConfig(beam=12.0, max_active=2000)
    res = lb.decode_batch(w, mats, cfg, want_lattice=False)
    tc, st, cnt = oracle_mod.decode_batch_mt(w, mats, 12.0, max_active=2000)
    assert all(st == 0)
    assert [r.total_cost for r in res] == tc.tolist()
    assert [[r.counters["n_tokens"], r.counters["n_scan"], r.counters["n_next"]] for r in res] == \
        [[c[0], c[1], c[6]] for c in cnt]


def test_c4_batched_mode_matches_lane_mode(oracle_mod, monkeypatch):
    """The 64-utterance C4 batch in both modes: identical costs and paths."""
    w = synthetic.hclg_graph(2, num_states=400_000, pool_size=6000, num_pdfs=600)
    mats = [synthetic.hclg_matrix(500 + i, num_frames=40, num_pdfs=600) for i in range(64)]
    cfg = lb.DecodeConfig(beam=13.0, max_active=2500)
    out = {}
    for mode in ("batched", "lane"):
        monkeypatch.setenv("LB_MODE", mode)
        out[mode] = lb.decode_batch(w, mats, cfg, want_lattice=False)
    assert [r.total_cost for r in out["batched"]] == [r.total_cost for r in out["lane"]]
    assert [r.words for r in out["batched"]] == [r.words for r in out["lane"]]
    tc, st, _ = oracle_mod.decode_batch_mt(w, mats, 13.0, max_active=2500)
    assert [r.total_cost for r in out["batched"]] == tc.tolist()


def test_larger_random_graphs(oracle_mod):
    for seed in range(9_000_000, 9_000_012):
        w, m = synthetic.random_task(seed, max_states=400, max_arcs=3000, num_labels=30,
                                     max_frames=60)
        got, ref = decode_both(w, m, oracle_mod, 7.0, 3.0)
        check_pair(got, ref, 3.0)


def test_w1_and_diamond_kats():
    w1 = lb.load_wfst_text("0 1 1 1 0.5\n0 2 2 2 1.0\n1 0.0\n2 0.0\n")
    c1 = lb.load_cost_matrix("1 2\n0.3 0.1\n")
    r = lb.decode_utterance(w1, c1, lb.DecodeConfig(keep_work_lattice=True))
    assert r.words == [1] and r.alignment == [(1, 0)] and not r.partial
    assert r.total_cost == pytest.approx(0.8)
    assert r.lattice.num_arcs == 2
    extras = {a.olabel: a.extra_cost for a in r.work_lattice.arcs()}
    assert extras[1] == pytest.approx(0.0, abs=1e-12) and extras[2] == pytest.approx(0.3, abs=1e-12)
    assert lb.decode_utterance(w1, c1, lb.DecodeConfig(lattice_beam=0.1)).lattice.num_arcs == 1
    assert lb.write_lattice_text(lb.decode_utterance(w1, c1, lb.DecodeConfig(lattice_beam=0.1)).lattice) \
        == "NODES 2 ARCS 1 START 0\nF 1 0.0\nA 0 1 1 1 0.5 0.3\n"
    dia = lb.load_wfst_text("0 1 1 1 0.1\n0 2 2 2 0.3\n1 3 1 0 0.2\n2 4 2 0 0.2\n"
                            "3 5 1 0 0.3\n4 5 2 0 0.3\n5 0.0\n")
    dc = lb.load_cost_matrix("3 2\n0.1 0.2\n0.1 0.2\n0.2 0.2\n")
    r = lb.decode_utterance(dia, dc, lb.DecodeConfig(lattice_beam=8.0, keep_work_lattice=True))
    assert r.total_cost == pytest.approx(1.0)
    by = {}
    for a in r.work_lattice.arcs():
        by.setdefault(a.ilabel, []).append(a.extra_cost)
    assert by[1] == pytest.approx([0.0] * 3, abs=1e-12) and by[2] == pytest.approx([0.4] * 3, abs=1e-12)
    assert lb.decode_utterance(dia, dc, lb.DecodeConfig(lattice_beam=0.39)).lattice.num_arcs == 3
    assert lb.decode_utterance(dia, dc, lb.DecodeConfig(lattice_beam=0.41)).lattice.num_arcs == 6


def test_error_paths():
    w1 = lb.load_wfst_text("0 1 1 1 0.5\n0 2 2 2 1.0\n1 0.0\n2 0.0\n")
    with pytest.raises(lb.DecodeFailure):
        lb.decode_utterance(w1, lb.load_cost_matrix("2 2\n0.3 0.1\n0.3 0.1\n"))
    with pytest.raises(lb.UsageError, match="label"):
        lb.decode_utterance(w1, lb.load_cost_matrix("1 1\n0.3\n"))
    part = lb.decode_utterance(lb.load_wfst_text("0 1 1 1 0.5\n2 0.0\n"), lb.load_cost_matrix("1 1\n0.3\n"))
    assert part.partial and part.words == [1] and part.total_cost == pytest.approx(0.8)
    g = synthetic.uniform_bench_graph(0, num_states=500, arcs_per_state=5, num_labels=40)
    m = synthetic.bench_matrix(1, num_frames=10, num_labels=40)
    with pytest.raises(lb.CapacityError) as e:
        lb.decode_utterance(g, m, lb.DecodeConfig(beam=13.0, max_tokens_per_frame=5))
    assert e.value.bound == "--max-tokens-per-frame"
    with pytest.raises(lb.CapacityError) as e:
        lb.decode_utterance(g, m, lb.DecodeConfig(beam=13.0, max_lattice_arcs=100))
    assert e.value.bound == "--max-lattice-arcs"


def test_expand_single_ops(oracle_mod):
    for seed in range(40):
        w, m = synthetic.random_task(seed)
        s, c, cut = lb.expand_emitting(w, np.array([w.start_state]), np.array([0.0]), m, 0, 6.0)
        rs, rc, rcut = oracle_mod.expand_emitting(w, [w.start_state], [0.0], m.costs[0], 6.0)
        assert np.array_equal(s, rs) and np.array_equal(c, rc) and (cut == rcut or
                                                                     (math.isinf(cut) and math.isinf(rcut)))
    chain = lb.load_wfst_text("0 1 0 0 0.3\n1 2 0 0 0.4\n2 0.0\n")
    s, c = lb.expand_nonemitting(chain, np.array([0]), np.array([0.5]), 100.0)
    assert s.tolist() == [0, 1, 2] and c == pytest.approx([0.5, 0.8, 1.2])
    s, c = lb.expand_nonemitting(chain, np.array([0]), np.array([0.5]), 1.0)
    assert s.tolist() == [0, 1]
    cyc = lb.load_wfst_text("0 1 0 0 0.0\n1 0 0 0 0.0\n0 0.0\n1 0.0\n")
    s, c = lb.expand_nonemitting(cyc, np.array([0]), np.array([0.2]), 100.0)
    assert s.tolist() == [0, 1] and c == pytest.approx([0.2, 0.2])
    for seed in range(40):
        w, _ = synthetic.random_task(seed)
        st = np.arange(0, w.num_states, 3)
        co = np.linspace(0.0, 2.0, len(st))
        s, c = lb.expand_nonemitting(w, st, co, 4.0)
        rs, rc = oracle_mod.expand_nonemitting(w, st, co, 4.0)
        assert np.array_equal(s, rs) and np.array_equal(c, rc)


@pytest.mark.parametrize("S,deg,L,beam,ma", [(2000, 5, 100, 10.0, 300), (3000, 4, 60, 12.0, 500)])
def test_max_active_uniform(oracle_mod, S, deg, L, beam, ma):
    w = synthetic.uniform_bench_graph(1, num_states=S, arcs_per_state=deg, num_labels=L)
    for u in range(3):
        m = synthetic.bench_matrix(300 + u, num_frames=30, num_labels=L)
        got, ref = decode_both(w, m, oracle_mod, beam, 6.0, max_active=ma)
        check_pair(got, ref, 6.0)


def test_config1_frames(oracle_mod):
    """Config C1 graph (uniform 10k x 5, 500 labels, beam 13), 2 utterances x 60 frames."""
    w = synthetic.config_graph("C1")
    for u in range(2):
        m = synthetic.bench_matrix(100 + u, num_frames=60, num_labels=500)
        got, ref = decode_both(w, m, oracle_mod, 13.0, 8.0, want_lattice=(u == 0))
        check_pair(got, ref, 8.0, want_lattice=(u == 0))


def test_hclg_with_epsilon_and_max_active(oracle_mod):
    w = synthetic.hclg_graph(3, num_states=300_000, pool_size=4000, num_pdfs=500)
    for u in range(2):
        m = synthetic.hclg_matrix(40 + u, num_frames=40, num_pdfs=500)
        got, ref = decode_both(w, m, oracle_mod, 13.0, 8.0, max_active=2000, want_lattice=(u == 0))
        check_pair(got, ref, 8.0, want_lattice=(u == 0))


def test_batch_equals_single(oracle_mod):
    w = synthetic.uniform_bench_graph(0, num_states=2000, arcs_per_state=5, num_labels=80)
    mats = [synthetic.bench_matrix(100 + i, num_frames=20 + 3 * i, num_labels=80) for i in range(10)]
    cfg = lb.DecodeConfig(beam=9.0, lattice_beam=2.0, lanes=3)
    bat = lb.decode_batch(w, mats, cfg)
    for m, b in zip(mats, bat):
        s = lb.decode_utterance(w, m, lb.DecodeConfig(beam=9.0, lattice_beam=2.0))
        assert s.words == b.words and s.total_cost == b.total_cost
        assert lb.write_lattice_text(s.lattice) == lb.write_lattice_text(b.lattice)
    tc, st, _ = oracle_mod.decode_batch_mt(w, mats, 9.0)
    assert all(st == 0) and [r.total_cost for r in bat] == tc.tolist()


def test_reference_wfst_object_duck_typing(oracle_mod):
    """Any object with the reference Wfst attributes decodes (drop-in)."""
    w, m = synthetic.random_task(5)

    class Duck:
        pass
    d = Duck()
    for k in ("num_states", "start_state", "arc_offsets", "arc_src", "arc_dst", "arc_ilabel",
              "arc_olabel", "arc_weight", "final_cost_array", "max_ilabel", "num_arcs"):
        setattr(d, k, getattr(w, k))
    r1 = lb.decode_utterance(d, m, lb.DecodeConfig(beam=8.0), want_lattice=False)
    r2 = lb.decode_utterance(w, m, lb.DecodeConfig(beam=8.0), want_lattice=False)
    assert r1.words == r2.words and r1.total_cost == r2.total_cost


def test_device_resident_and_zero_copy_paths_agree(oracle_mod, monkeypatch):
    """The three ways costs reach the kernel give identical results: device-resident
    tensors (lb_decode_batch_device, the bench's `value` path), host numpy through
    pinned zero-copy rows (the default 1-best e2e path), and host numpy copied to
    HBM first (LB_E2E_COPY=1).  All equal the oracle."""
    import torch

    from paper_1804_03243_b200.resident import decode_batch_resident
    w = synthetic.hclg_graph(7, num_states=200_000, pool_size=3000, num_pdfs=400)
    mats = [np.ascontiguousarray(synthetic.hclg_matrix(60 + i, num_frames=25 + 5 * i, num_pdfs=400).costs)
            for i in range(6)]
    cfg = lb.DecodeConfig(beam=12.0, max_active=1500)
    tc, st, _ = oracle_mod.decode_batch_mt(w, mats, 12.0, max_active=1500)
    assert all(st == 0)
    monkeypatch.setenv("LB_ZC_MIN", "1")   # zero-copy even for a batch this small
    zc = lb.decode_batch(w, mats, cfg, want_lattice=False)
    monkeypatch.setenv("LB_E2E_COPY", "1")
    cp = lb.decode_batch(w, mats, cfg, want_lattice=False)
    monkeypatch.delenv("LB_E2E_COPY")
    outs, _ = decode_batch_resident(w, [torch.from_numpy(m.copy()).cuda() for m in mats], cfg)
    assert [r.total_cost for r in zc] == tc.tolist()
    assert [r.total_cost for r in cp] == tc.tolist()
    assert [o["total_cost"] for o in outs] == tc.tolist()
    for r, o in zip(zc, outs):
        il = w.arc_ilabel[o["path"]]
        assert r.alignment == list(zip(il[il > 0].tolist(), range(int((il > 0).sum()))))


def test_results_outlive_later_decodes():
    """C-ABI results own their final lattices: a result held across later decodes
    (which reuse the pinned D2H arena once no result points into it) still reads
    back the lattice it was decoded with."""
    import ctypes as C

    from paper_1804_03243_b200 import _lib
    from paper_1804_03243_b200 import decoder as dec
    w = synthetic.uniform_bench_graph(3, num_states=3000, arcs_per_state=5, num_labels=100)
    sets = [[np.ascontiguousarray(synthetic.bench_matrix(100 * k + i, num_frames=60, num_labels=100).costs)
             for i in range(3)] for k in range(3)]
    cfg = lb.DecodeConfig(beam=10.0, lattice_beam=5.0)
    want = [lb.decode_batch(w, mats, cfg) for mats in sets]
    L = _lib.lib()
    g = dec.device_graph(w, 0)

    def raw(mats):
        n = len(mats)
        cptrs = (_lib.PD * n)(*[m.ctypes.data_as(_lib.PD) for m in mats])
        T = np.asarray([m.shape[0] for m in mats], dtype=np.int32)
        c = cfg.to_c(True, False)
        res = _lib.PV()
        assert L.lb_decode_batch(g.handle, n, cptrs, T.ctypes.data_as(_lib.P32), 100, C.byref(c),
                                 C.byref(res)) == 0
        return res

    held = [raw(mats) for mats in sets]          # all three alive at once
    for k in (1, 0, 2):
        for u in range(3):
            assert dec._final_lattice(held[k], u, 60).same_lattice(want[k][u].lattice), (k, u)
        L.lb_result_free(held[k])
        held[k] = raw(sets[(k + 1) % 3])         # a decode after a free reuses the arena
        for u in range(3):
            assert dec._final_lattice(held[k], u, 60).same_lattice(want[(k + 1) % 3][u].lattice)
    for r in held:
        L.lb_result_free(r)


@pytest.mark.parametrize("D", [2000, 1999])
def test_progressive_zero_copy_staging(oracle_mod, monkeypatch, D):
    """Lane-kernel 1-best decodes of host numpy costs stage the rows progressively
    (frame chunks published through a mapped counter while the kernel runs).
    Repeated calls through the same staging buffer with new data and ragged
    lengths, multi-threaded staging (> 8 MB), and the non-progressive path all
    equal the oracle bit-exactly."""
    monkeypatch.setenv("LB_MODE", "lane")
    monkeypatch.setenv("LB_ZC_MIN", "1")
    w = synthetic.hclg_graph(8, num_states=200_000, pool_size=3000, num_pdfs=D)
    cfg = lb.DecodeConfig(beam=12.0, max_active=1500)
    for rnd in range(5):
        mats = [np.ascontiguousarray(synthetic.hclg_matrix(900 + 10 * rnd + i, num_frames=120 + 37 * i + rnd,
                                                           num_pdfs=D).costs) for i in range(8)]
        assert sum(m.nbytes for m in mats) > (8 << 20)
        tc, st, _ = oracle_mod.decode_batch_mt(w, mats, 12.0, max_active=1500)
        assert all(st == 0)
        if rnd == 4:
            monkeypatch.setenv("LB_NO_PROGRESSIVE", "1")
        res = lb.decode_batch(w, mats, cfg, want_lattice=False)
        assert [r.total_cost for r in res] == tc.tolist(), rnd
    monkeypatch.delenv("LB_NO_PROGRESSIVE")


@pytest.mark.parametrize("ctas", [2, 8])
def test_racecheck_lane_kernel(ctas):
    """racecheck finds no shared-memory hazard in the persistent-lane kernel
    (tiny 1-best with progressive staging, and lattice decodes; 2- and 8-CTA
    clusters).  It caught a barrier-divergence race in the staging wait."""
    import os
    import shutil
    import subprocess
    import sys
    cs = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(cs):
        pytest.skip("compute-sanitizer not installed")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = subprocess.run([cs, "--tool", "racecheck", "--error-exitcode", "9", sys.executable,
                          os.path.join(root, "tools", "racecheck_lane.py"), str(ctas)],
                         capture_output=True, text=True, timeout=900)
    out = res.stdout + res.stderr
    assert res.returncode == 0, out[-6000:]
    assert "ok %d" % ctas in res.stdout and "RACECHECK SUMMARY: 0 hazards displayed (0 errors" in out, out[-3000:]


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_compute_sanitizer_clean(tool):
    """compute-sanitizer finds no memory error, shared-memory race or barrier misuse
    in small 1-best + lattice decodes with epsilon arcs and max-active:
    the batched mode and, except under racecheck (over 20 minutes on the lane
    kernels' shared memory), 16-CTA lanes reading progressively staged host rows and
    2-CTA lanes with lattices."""
    import os
    import shutil
    import subprocess
    import sys
    cs = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(cs):
        pytest.skip("compute-sanitizer not installed")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    prog = (
        "import sys; sys.path.insert(0, %r)\n"
        "import paper_1804_03243_b200 as lb\n"
        "from paper_1804_03243_b200 import synthetic\n"
        "import os; os.environ['LB_MODE'] = 'batched'\n"
        "w = synthetic.hclg_graph(5, num_states=20000, pool_size=500, num_pdfs=100)\n"
        "ms = [synthetic.hclg_matrix(9 + i, num_frames=6, num_pdfs=100) for i in range(2)]\n"
        "r = lb.decode_batch(w, ms, lb.DecodeConfig(beam=10.0, lattice_beam=3.0, max_active=300))\n"
        "q = lb.decode_batch(w, ms, lb.DecodeConfig(beam=10.0, max_active=300), want_lattice=False)\n"
        "assert [x.total_cost for x in r] == [x.total_cost for x in q]\n"
        "if %r:\n"
        "    m6 = [synthetic.hclg_matrix(30 + i, num_frames=5, num_pdfs=100) for i in range(6)]\n"
        "    del os.environ['LB_MODE']; os.environ['LB_ZC_MIN'] = '1'\n"
        "    q6 = lb.decode_batch(w, m6, lb.DecodeConfig(beam=10.0, max_active=300), want_lattice=False)\n"
        "    os.environ['LB_MODE'] = 'lane'\n"
        "    l6 = lb.decode_batch(w, m6, lb.DecodeConfig(beam=10.0, lattice_beam=3.0, max_active=300))\n"
        "    assert [x.total_cost for x in q6] == [x.total_cost for x in l6]\n"
        "print('ok', [x.total_cost for x in r])\n" % (root, tool != "racecheck"))
    res = subprocess.run([cs, "--tool", tool, "--error-exitcode", "9", sys.executable, "-c", prog],
                         capture_output=True, text=True, timeout=1200)
    out = res.stdout + res.stderr
    assert res.returncode == 0, out[-6000:]
    clean = "ERROR SUMMARY: 0 errors" in out or "RACECHECK SUMMARY: 0 hazards displayed (0 errors" in out
    assert "ok" in res.stdout and clean, out[-3000:]


A4_GRAPH = "3 1 1 1 1.0\n3 2 1 2 1.0000000000009095\n1 2 0 0 0.0\n2 1 0 0 0.0\n1 0.0\n2 0.0\n"


@pytest.mark.parametrize("mode", ["batched", "lane"])
@pytest.mark.parametrize("want_lattice", [False, True])
def test_backtrace_cycle_raises_on_device(oracle_mod, monkeypatch, mode, want_lattice):
    """states 1 and 2 end up as each other's epsilon
    predecessor (f32-equal costs, lower arc ids win the ties), so the reference's
    _backtrace never terminates.  The device walk is step-bounded and reports
    InternalInvariantError, as the oracle does."""
    monkeypatch.setenv("LB_MODE", mode)
    w = lb.load_wfst_text(A4_GRAPH)
    m = lb.load_cost_matrix("1 1\n0.0\n")
    ref = oracle_mod.decode(w, m, 10.0, want_lattice=False)
    assert ref.status == 4 and "backtrace" in ref.message
    with pytest.raises(lb.InternalInvariantError, match="backtrace"):
        lb.decode_utterance(w, m, lb.DecodeConfig(beam=10.0), want_lattice=want_lattice)
    # the graph stays usable afterwards (the error path reset its lane state)
    ok = lb.load_wfst_text("0 1 1 1 0.5\n0 2 2 2 1.0\n1 0.0\n2 0.0\n")
    r = lb.decode_utterance(ok, lb.load_cost_matrix("1 2\n0.3 0.1\n"), lb.DecodeConfig())
    assert r.words == [1]


@pytest.mark.parametrize("mode", ["batched", "lane"])
def test_shorter_batch_after_longer_batch(oracle_mod, monkeypatch, mode):
    """A workspace grown by a batch of long utterances is reused by a later batch of
    shorter ones: every lane's best path (words, alignment) still matches the
    oracle (the path buffer stride is the workspace's, not the call's)."""
    monkeypatch.setenv("LB_MODE", mode)
    w = synthetic.hclg_graph(6, num_states=100_000, pool_size=2000, num_pdfs=300)
    cfg = lb.DecodeConfig(beam=12.0, max_active=800)
    for T, n in ((160, 12), (40, 12), (90, 5), (25, 12)):
        mats = [synthetic.hclg_matrix(3000 + 100 * T + i, num_frames=T - (i % 3), num_pdfs=300)
                for i in range(n)]
        res = lb.decode_batch(w, mats, cfg, want_lattice=False)
        for m, r in zip(mats, res):
            ref = oracle_mod.decode(w, m, 12.0, max_active=800, want_lattice=False, collect_frames=False)
            assert ref.ok
            assert r.words == ref.words and r.alignment == ref.alignment, (T, n)
            assert r.total_cost == ref.total_cost


def test_epsilon_round_tags_reset(oracle_mod, monkeypatch):
    """Round tags are reset (LB_FORCE_TAG_RESET forces it after every decode);
    decodes before and after a reset equal the oracle."""
    monkeypatch.setenv("LB_FORCE_TAG_RESET", "1")
    w = synthetic.hclg_graph(3, num_states=50_000, pool_size=1500, num_pdfs=200)
    cfg = lb.DecodeConfig(beam=12.0, max_active=600)
    for k in range(3):
        mats = [synthetic.hclg_matrix(4000 + 10 * k + i, num_frames=30, num_pdfs=200) for i in range(6)]
        res = lb.decode_batch(w, mats, cfg, want_lattice=False)
        tc, st, _ = oracle_mod.decode_batch_mt(w, mats, 12.0, max_active=600)
        assert all(st == 0) and [r.total_cost for r in res] == tc.tolist()


def _ragged_batch(n, seed0, num_pdfs=300, tmin=8, tmax=70):
    rng = np.random.default_rng(seed0)
    return [np.ascontiguousarray(synthetic.hclg_matrix(seed0 + i, num_frames=int(rng.integers(tmin, tmax + 1)),
                                                       num_pdfs=num_pdfs).costs) for i in range(n)]


@pytest.mark.parametrize("slots,zc", [(0, False), (1, False), (3, False), (0, True), (3, True)])
def test_refilling_lanes_streamed_ring(oracle_mod, monkeypatch, slots, zc):
    """A ragged batch much larger than the lane count: one launch, lanes refill
    from the longest-first job queue, host rows stream through the pinned ring
    (LB_RING_SLOTS forces heavy slot reuse: every slot is rewritten many times
    inside one kernel), copied slot by slot into a device ring on a copy stream
    (default) or read zero-copy over PCIe (LB_RING_ZC).  Every utterance equals
    the oracle, in input order."""
    if slots:
        monkeypatch.setenv("LB_RING_SLOTS", str(slots))
    if zc:
        monkeypatch.setenv("LB_RING_ZC", "1")
    w = synthetic.hclg_graph(9, num_states=60_000, pool_size=1500, num_pdfs=300)
    mats = _ragged_batch(90, 7000 + slots)
    cfg = lb.DecodeConfig(beam=12.0, max_active=600, lanes=6)
    res = lb.decode_batch(w, mats, cfg, want_lattice=False)
    tc, st, cnt = oracle_mod.decode_batch_mt(w, mats, 12.0, max_active=600)
    assert all(st == 0)
    assert [r.total_cost for r in res] == tc.tolist()
    assert [[r.counters["n_tokens"], r.counters["n_scan"], r.counters["n_next"]] for r in res] == \
        [[c[0], c[1], c[6]] for c in cnt]
    for i in (0, 17, 89):
        ref = oracle_mod.decode(w, mats[i], 12.0, max_active=600, want_lattice=False, collect_frames=False)
        assert res[i].words == ref.words and res[i].alignment == ref.alignment


def test_refilling_lanes_device_resident(oracle_mod):
    """The same queue with HBM-resident costs (lb_decode_batch_device)."""
    import torch

    from paper_1804_03243_b200.resident import decode_batch_resident
    w = synthetic.hclg_graph(9, num_states=60_000, pool_size=1500, num_pdfs=300)
    mats = _ragged_batch(70, 7100)
    cfg = lb.DecodeConfig(beam=12.0, max_active=600, lanes=5)
    outs, _ = decode_batch_resident(w, [torch.from_numpy(m.copy()).cuda() for m in mats], cfg)
    tc, st, _ = oracle_mod.decode_batch_mt(w, mats, 12.0, max_active=600)
    assert all(st == 0) and [o["total_cost"] for o in outs] == tc.tolist()
    assert all(o["status"] == 0 for o in outs)


def test_refill_and_waves_agree(monkeypatch):
    """Refilling lanes (default) and static waves (LB_NO_REFILL) give identical results."""
    w = synthetic.hclg_graph(10, num_states=60_000, pool_size=1500, num_pdfs=300)
    mats = _ragged_batch(40, 7200)
    cfg = lb.DecodeConfig(beam=12.0, max_active=600, lanes=4)
    a = lb.decode_batch(w, mats, cfg, want_lattice=False)
    monkeypatch.setenv("LB_NO_REFILL", "1")
    b = lb.decode_batch(w, mats, cfg, want_lattice=False)
    assert [(r.total_cost, r.words, r.alignment) for r in a] == [(r.total_cost, r.words, r.alignment) for r in b]


def test_multi_device_replicas_on_one_gpu(oracle_mod):
    """decode_batch(devices=[0, 0]): two independent replicas of the graph on
    device 0, LPT shards on two host threads (lb_decode_batch_multi), results in
    input order equal to the single-replica decode and the oracle."""
    w = synthetic.hclg_graph(11, num_states=60_000, pool_size=1500, num_pdfs=300)
    mats = _ragged_batch(30, 7300)
    one = lb.decode_batch(w, mats, lb.DecodeConfig(beam=12.0, max_active=600), want_lattice=False)
    two = lb.decode_batch(w, mats, lb.DecodeConfig(beam=12.0, max_active=600, devices=(0, 0)),
                          want_lattice=False)
    assert [(r.total_cost, r.words) for r in one] == [(r.total_cost, r.words) for r in two]
    tc, st, _ = oracle_mod.decode_batch_mt(w, mats, 12.0, max_active=600)
    assert [r.total_cost for r in two] == tc.tolist()
    lat = lb.decode_batch(w, mats[:6], lb.DecodeConfig(beam=12.0, lattice_beam=4.0, max_active=600,
                                                       devices=(0, 0)))
    single = lb.decode_batch(w, mats[:6], lb.DecodeConfig(beam=12.0, lattice_beam=4.0, max_active=600))
    assert all(a.lattice.same_lattice(b.lattice) for a, b in zip(lat, single))


def _work_arrays(lat):
    from paper_1804_03243_b200.lattice import STATUS_LIVE
    frames = [f.costs.copy() for f in lat.frames]
    blocks = []
    for b in range(len(lat.frames)):
        a = lat.block_arrays(b)
        blocks.append({"from_idx": a["from_idx"].astype(np.int64), "to_idx": a["to_idx"].astype(np.int64),
                       "ilabel": a["ilabel"], "graph_cost": a["graph_cost"].copy(),
                       "acoustic_cost": a["acoustic_cost"].copy(),
                       "status": np.where(a["status"] == STATUS_LIVE, 0, 1).astype(np.uint8),
                       "extra": a["extra"].copy()})
    return frames, blocks


def test_prune_lattice_single_op(oracle_mod):
    """prune_lattice (lattice.py:365-431) on the device: re-pruning a decoded
    work lattice with its own beam and final costs is idempotent (the reference's
    test_reprune_is_idempotent); a tighter beam, and mid-decode prunes from an
    earlier frontier with a zero terminus, match the CPU restatement
    (oracle/prune_oracle.py) arc by arc (status exactly, extras within 1e-9)."""
    from oracle import prune_oracle as PO
    from paper_1804_03243_b200.lattice import STATUS_LIVE
    rng = np.random.default_rng(5)
    checked = 0
    for seed in range(15_000_000, 15_000_025):
        w, m = synthetic.random_task(seed, allow_eps_cycles=seed % 2 == 1)
        try:
            r = lb.decode_utterance(w, m, lb.DecodeConfig(beam=9.0, lattice_beam=5.0, keep_work_lattice=True))
        except lb.LatbeamError:
            continue
        lat = r.work_lattice
        before = lat.live_arc_table(include_pruned=True)
        lb.prune_lattice(lat, lat.frames[-1], 5.0, final_costs=lat.final_token_costs)
        after = lat.live_arc_table(include_pruned=True)
        assert np.array_equal(before["status"], after["status"])
        assert np.allclose(before["extra"], after["extra"], equal_nan=True)
        for _ in range(2):
            t = int(rng.integers(0, len(lat.frames)))
            beam = float(rng.uniform(0.0, 5.0))
            fc = lat.final_token_costs if t == len(lat.frames) - 1 and not r.partial else None
            frames, blocks = _work_arrays(lat)
            if fc is None:
                term = np.zeros(len(frames[t]))
            else:
                tot = frames[t] + fc
                term = tot - tot.min()
            want, want_ne = PO.prune(frames, blocks, t, beam, term)
            lb.prune_lattice(lat, lat.frames[t], beam, final_costs=fc)
            for b in range(t + 1):
                got = lat.block_arrays(b)
                st = np.where(got["status"] == STATUS_LIVE, 0, 1)
                assert np.array_equal(st, want[b]["status"]), (seed, t, b)
                fin = np.isfinite(want[b]["extra"])
                assert np.array_equal(np.isfinite(got["extra"]), fin)
                assert np.allclose(got["extra"][fin], want[b]["extra"][fin], rtol=0, atol=1e-9)
                assert np.allclose(lat.node_extra[b], want_ne[b], rtol=0, atol=1e-9, equal_nan=True) or \
                    np.array_equal(np.isinf(lat.node_extra[b]), np.isinf(want_ne[b]))
            checked += 1
    assert checked >= 20
    with pytest.raises(lb.UsageError):
        lb.prune_lattice(lat, lat.frames[0], -1.0)
    with pytest.raises(lb.UsageError):
        lb.prune_lattice(lat, type(lat.frames[0])(0, lat.frames[0].states, lat.frames[0].costs,
                                                  lat.frames[0].pred_arc, lat.frames[0].pred_idx), 1.0)


@pytest.mark.parametrize("widen", [False, True])
def test_f32_device_costs_equal_widened_decode(oracle_mod, monkeypatch, widen):
    """f32 HBM-resident log-likelihoods decode exactly like the f64-widened
    matrices: fused widening at the row load (refilling lanes) and the HBM
    widening pass (LB_F32_WIDEN, every other mode), both vs the oracle."""
    import torch

    from paper_1804_03243_b200.resident import decode_batch_resident
    if widen:
        monkeypatch.setenv("LB_F32_WIDEN", "1")
    w = synthetic.hclg_graph(12, num_states=60_000, pool_size=1500, num_pdfs=300)
    m32 = [np.ascontiguousarray(m.astype(np.float32)) for m in _ragged_batch(40, 7400)]
    wide = [m.astype(np.float64) for m in m32]
    cfg = lb.DecodeConfig(beam=12.0, max_active=600, lanes=6)
    outs, _ = decode_batch_resident(w, [torch.from_numpy(m).cuda() for m in m32], cfg)
    tc, st, _ = oracle_mod.decode_batch_mt(w, wide, 12.0, max_active=600)
    assert all(st == 0) and [o["total_cost"] for o in outs] == tc.tolist()
    host = lb.decode_batch(w, wide, cfg, want_lattice=False)
    for o, r in zip(outs, host):
        il = w.arc_ilabel[o["path"]]
        assert r.alignment == list(zip(il[il > 0].tolist(), range(int((il > 0).sum()))))


def test_work_lattice_by_default():
    """DecodeResult.work_lattice exists whenever a lattice is requested
    (decoder.py:605-606): a LazyWorkLattice that materialises on first use and
    equals the eagerly kept one; 1-best decodes have none."""
    from paper_1804_03243_b200.lattice import WorkLattice
    w, m = synthetic.random_task(21, allow_eps_cycles=True)
    lazy = lb.decode_utterance(w, m, lb.DecodeConfig(beam=9.0, lattice_beam=4.0))
    eager = lb.decode_utterance(w, m, lb.DecodeConfig(beam=9.0, lattice_beam=4.0, keep_work_lattice=True))
    assert isinstance(lazy.work_lattice, WorkLattice)
    a = lazy.work_lattice.live_arc_table(include_pruned=True)
    b = eager.work_lattice.live_arc_table(include_pruned=True)
    assert set(a) == set(b) and all(np.array_equal(a[k], b[k]) for k in a)
    assert lazy.work_lattice.num_frames == eager.work_lattice.num_frames
    assert [f.states.tolist() for f in lazy.work_lattice.frames] == [f.states.tolist() for f in eager.work_lattice.frames]
    assert lb.decode_utterance(w, m, lb.DecodeConfig(beam=9.0), want_lattice=False).work_lattice is None


def test_row_prefetch_and_its_fallbacks(oracle_mod, monkeypatch):
    """The next-frame row prefetch (16-byte cp.async of f64 rows) and the paths
    that cannot use it -- matrices only 8-byte aligned in HBM, LB_NO_ROWPF --
    all equal the oracle."""
    import torch

    from paper_1804_03243_b200.resident import decode_batch_resident
    w = synthetic.hclg_graph(13, num_states=60_000, pool_size=1500, num_pdfs=300)
    mats = _ragged_batch(24, 7500)
    tc, st, _ = oracle_mod.decode_batch_mt(w, mats, 12.0, max_active=600)
    assert all(st == 0)
    cfg = lb.DecodeConfig(beam=12.0, max_active=600, lanes=5)
    aligned = [torch.from_numpy(m.copy()).cuda() for m in mats]
    flat = torch.zeros(sum(m.size for m in mats) + 1, dtype=torch.float64, device="cuda")
    views, o = [], 1                                     # every matrix starts 8 bytes off a 16-byte line
    for m in mats:
        v = flat[o:o + m.size].view(m.shape)
        v.copy_(torch.from_numpy(m))
        views.append(v)
        o += m.size
    for tens in (aligned, views):
        outs, _ = decode_batch_resident(w, tens, cfg)
        assert [x["total_cost"] for x in outs] == tc.tolist()
    monkeypatch.setenv("LB_NO_ROWPF", "1")
    outs, _ = decode_batch_resident(w, aligned, cfg)
    assert [x["total_cost"] for x in outs] == tc.tolist()


def test_finalize_lattice_single_op():
    """finalize_lattice (lattice.py:537-598) on the device for a work lattice:
    equal to the decode's own device-finalised lattice, to the numpy restatement
    (oracle/finalize_oracle.py) after a re-prune at a tighter beam, and the
    reference's DecodeFailure when nothing survives."""
    from oracle import finalize_oracle as FO
    n = 0
    for seed in range(16_000_000, 16_000_020):
        w, m = synthetic.random_task(seed, allow_eps_cycles=seed % 2 == 0)
        try:
            r = lb.decode_utterance(w, m, lb.DecodeConfig(beam=9.0, lattice_beam=4.0, keep_work_lattice=True))
        except lb.LatbeamError:
            continue
        lat = r.work_lattice
        fl = lb.finalize_lattice(lat)
        assert fl.same_lattice(r.lattice)
        assert np.array_equal(fl.node_frame, r.lattice.node_frame) and np.array_equal(fl.node_idx, r.lattice.node_idx)
        lb.prune_lattice(lat, lat.frames[-1], 1.0, final_costs=None if r.partial else lat.final_token_costs)
        try:
            want = FO.finalize(lat.live_arc_table(), lat.start_idx, lat.num_frames, lat.partial, lat.final_token_costs)
        except ValueError as exc:
            with pytest.raises(lb.DecodeFailure, match=str(exc)):
                lb.finalize_lattice(lat)
            continue
        got = lb.finalize_lattice(lat)
        assert got.num_nodes == want["num_nodes"] and got.start == want["start"]
        for k in ("final_ids", "final_costs", "from_", "to", "ilabel", "olabel", "graph_cost", "acoustic_cost",
                  "node_frame", "node_idx"):
            assert np.array_equal(getattr(got, k), want[k]), k
        n += 1
    assert n >= 10


@pytest.mark.parametrize("tool", ["memcheck", "synccheck"])
def test_compute_sanitizer_round2_paths(tool):
    """compute-sanitizer on the round-2 paths: refilling lanes fed through the
    streamed ring with slot reuse (8 jobs, 2 lanes, 3 slots) and the row prefetch,
    mixed-width launches, HBM-resident f32 rows, two replicas on one device, and
    the prune_lattice / finalize_lattice single ops."""
    import os
    import shutil
    import subprocess
    import sys
    cs = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(cs):
        pytest.skip("compute-sanitizer not installed")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    prog = (
        "import sys, os; sys.path.insert(0, %r)\n"
        "import numpy as np, torch\n"
        "import paper_1804_03243_b200 as lb\n"
        "from paper_1804_03243_b200 import synthetic\n"
        "from paper_1804_03243_b200.resident import decode_batch_resident\n"
        "w = synthetic.hclg_graph(5, num_states=20000, pool_size=500, num_pdfs=100)\n"
        "ms = [np.ascontiguousarray(synthetic.hclg_matrix(40 + i, num_frames=4 + i, num_pdfs=100).costs) for i in range(8)]\n"
        "os.environ['LB_RING_SLOTS'] = '3'\n"
        "os.environ['LB_MODE'] = 'lane'\n"
        "a = lb.decode_batch(w, ms, lb.DecodeConfig(beam=10.0, max_active=300, lanes=2), want_lattice=False)\n"
        "os.environ['LB_MIXED_N3'] = '1'\n"
        "b = lb.decode_batch(w, ms, lb.DecodeConfig(beam=10.0, max_active=300, lanes=2), want_lattice=False)\n"
        "del os.environ['LB_MIXED_N3']; del os.environ['LB_MODE']\n"
        "f = decode_batch_resident(w, [torch.from_numpy(m.astype(np.float32)).cuda() for m in ms],\n"
        "                          lb.DecodeConfig(beam=10.0, max_active=300, lanes=2))[0]\n"
        "c = lb.decode_batch(w, ms[:4], lb.DecodeConfig(beam=10.0, max_active=300, devices=(0, 0)), want_lattice=False)\n"
        "assert [x.total_cost for x in a] == [x.total_cost for x in b]\n"
        "assert [x.total_cost for x in a[:4]] == [x.total_cost for x in c]\n"
        "assert all(o['status'] == 0 for o in f)\n"
        "t, m = synthetic.random_task(21, allow_eps_cycles=True)\n"
        "r = lb.decode_utterance(t, m, lb.DecodeConfig(beam=9.0, lattice_beam=4.0, keep_work_lattice=True))\n"
        "lat = r.work_lattice\n"
        "assert lb.finalize_lattice(lat).same_lattice(r.lattice)\n"
        "lb.prune_lattice(lat, lat.frames[-1], 1.0, final_costs=None if r.partial else lat.final_token_costs)\n"
        "print('ok', [x.total_cost for x in a])\n" % root)
    res = subprocess.run([cs, "--tool", tool, "--error-exitcode", "9", sys.executable, "-c", prog],
                         capture_output=True, text=True, timeout=1500)
    out = res.stdout + res.stderr
    assert res.returncode == 0, out[-6000:]
    assert "ok" in res.stdout and "ERROR SUMMARY: 0 errors" in out, out[-3000:]
