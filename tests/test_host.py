"""Host-side pieces that need no GPU: formats, packing, config validation,
generators, and the oracle on the reference's hand-sized known-answer tests."""

import math

import numpy as np
import pytest

import paper_1804_03243_b200 as lb
from paper_1804_03243_b200 import packing, synthetic

W1 = "0 1 1 1 0.5\n0 2 2 2 1.0\n1 0.0\n2 0.0\n"
DIAMOND = ("0 1 1 1 0.1\n0 2 2 2 0.3\n1 3 1 0 0.2\n2 4 2 0 0.2\n3 5 1 0 0.3\n4 5 2 0 0.3\n5 0.0\n")


class TestPacking:
    def test_known_words(self):          # test_packing.py:8-15
        assert lb.pack(0.0, 5) == 0x8000000000000005
        assert lb.pack(1.0, 3) < lb.pack(1.0, 7) < lb.pack(1.5, 0)

    def test_order_and_roundtrip(self):
        rng = np.random.default_rng(0)
        c = np.concatenate([rng.uniform(-5, 5, 500), [0.0, -0.0, 1e-30, -1e-30]])
        a = rng.integers(0, 2 ** 32, len(c))
        w = packing.pack_array(c, a)
        key = sorted(range(len(c)), key=lambda i: (np.float32(c[i]), a[i]))
        assert np.all(np.diff(w[key].astype(np.float64)) >= 0)
        cc, aa = packing.unpack_array(w)
        assert np.array_equal(aa, a) and np.array_equal(cc, c.astype(np.float32).astype(np.float64))

    def test_cost64(self):
        for x in (-3.5, 0.0, 1e-300, 7.25, math.inf):
            assert packing.decode_cost64(packing.encode_cost64(x)) == x
        assert packing.encode_cost64(-1.0) < packing.encode_cost64(0.5) < packing.encode_cost64(math.inf)

    def test_rejects(self):
        with pytest.raises(lb.UsageError):
            lb.pack(-1.0, 0)
        with pytest.raises(lb.UsageError):
            lb.pack(1.0, 2 ** 32)
        with pytest.raises(lb.UsageError):
            lb.unpack(int(lb.SENTINEL))


class TestFormats:
    def test_wfst_roundtrip_and_layout(self):
        w = lb.load_wfst_text(DIAMOND)
        assert w.num_states == 6 and w.num_arcs == 6 and w.start_state == 0
        assert w.out_arc_range(0) == (0, 2)
        assert lb.write_wfst_text(lb.load_wfst_text(lb.write_wfst_text(w))) == lb.write_wfst_text(w)
        for seed in range(50):
            g = synthetic.random_wfst(np.random.default_rng(seed))
            s1 = lb.write_wfst_text(g)
            assert lb.write_wfst_text(lb.load_wfst_text(s1)) == s1

    @pytest.mark.parametrize("text,exc", [("0 1 1\n", lb.ParseError), ("0 1 1 1 -1\n1 0\n", lb.ValidationError),
                                          ("1 0.0\n", lb.ValidationError), ("0 1 1 1 0.5\n", lb.ValidationError),
                                          ("0 1 x 1\n1\n", lb.ParseError)])
    def test_wfst_errors(self, text, exc):
        with pytest.raises(exc):
            lb.load_wfst_text(text)

    def test_cost_matrix(self):
        m = lb.load_cost_matrix("2 2\n0.1 0.2\n0.3 0.4\n")
        assert m.num_frames == 2 and m.num_labels == 2
        assert lb.load_cost_matrix(lb.write_cost_matrix(m)).costs.tolist() == m.costs.tolist()
        assert lb.acoustic_cost(m, 1, 2, 0.5) == pytest.approx(0.2)
        for bad in ("", "2 2\n0.1 0.2\n", "1 2\n0.1 nan\n", "1 2\n0.1\n"):
            with pytest.raises(lb.ParseError):
                lb.load_cost_matrix(bad)
        with pytest.raises(lb.UsageError):
            lb.CostMatrix(np.array([[np.inf]]))

    def test_lattice_text(self):
        fl = lb.FinalLattice(2, 0, np.array([1]), np.array([0.0]), np.array([0]), np.array([1]),
                             np.array([1]), np.array([1]), np.array([0.5]), np.array([0.3]))
        t = lb.write_lattice_text(fl)
        assert t == "NODES 2 ARCS 1 START 0\nF 1 0.0\nA 0 1 1 1 0.5 0.3\n"
        assert lb.write_lattice_text(lb.read_lattice_text(t)) == t
        for bad in ("", "NODES 2 ARCS 2 START 0\nA 0 1 1 1 0.5 0.3\n", "NODES 1 ARCS 1 START 0\nA 0 1 1 1 0.5 0.3\n",
                    "NODES 2 ARCS 0 START 0\nX 1\n"):
            with pytest.raises(lb.ParseError):
                lb.read_lattice_text(bad)

    def test_native_text_writer_matches_python_repr(self):
        """lb_lattice_text (native, threaded) == the pure-Python writer, byte for byte,
        over awkward floats (repr switches to exponent form at 1e-4 / 1e16, keeps
        '.0' on integral values, shortest round-trip digits) and a big lattice."""
        from paper_1804_03243_b200.lattice import write_lattice_text_py
        vals = np.array([0.0, -0.0, 1.0, 100.0, 0.1, 1 / 3, 1e-4, 1e-5, 9.999e-5, 1e15, 1e16, 123456.789,
                         2.5e-300, 1.7976931348623157e308, 5e-324, 0.30000000000000004, 7.0e22, -3.25])
        n = len(vals)
        fl = lb.FinalLattice(n + 1, 0, np.array([n]), np.array([vals[3]]), np.arange(n), np.arange(1, n + 1),
                             np.arange(n) % 7, np.arange(n) % 5, vals, vals[::-1].copy())
        assert lb.write_lattice_text(fl) == write_lattice_text_py(fl)
        rng = np.random.default_rng(3)
        m = 200_000
        big = lb.FinalLattice(m + 1, 0, np.array([m, m - 1]), rng.uniform(0, 3, 2), np.arange(m),
                              np.arange(1, m + 1), rng.integers(0, 3000, m), rng.integers(0, 30000, m),
                              rng.uniform(0, 3, m), rng.uniform(-5, 5, m) * 10.0 ** rng.integers(-8, 8, m))
        assert lb.write_lattice_text(big) == write_lattice_text_py(big)

    def test_npz_roundtrip(self, tmp_path):
        w = synthetic.hclg_graph(1, num_states=5000, pool_size=200)
        p = tmp_path / "g.npz"
        lb.save_wfst_npz(w, p)
        v = lb.load_wfst_npz(p)
        for k in ("arc_offsets", "arc_dst", "arc_ilabel", "arc_olabel", "arc_weight", "final_cost_array"):
            assert np.array_equal(getattr(w, k), getattr(v, k))


class TestConfig:
    def test_defaults_match_reference(self):        # test_decoder.py:189-195
        c = lb.DecodeConfig()
        assert (c.beam, c.lattice_beam, c.num_shards, c.group_size, c.prune_interval) == (14.0, 8.0, 32, 32, 25)
        assert c.max_active == 0
        c.validate()

    @pytest.mark.parametrize("field,value", [("beam", 0.0), ("beam", math.inf), ("lattice_beam", -0.5),
                                             ("acoustic_scale", 0.0), ("num_workers", 0), ("num_shards", 0),
                                             ("prune_interval", 0), ("scheduler", "roundrobin"),
                                             ("max_active", -1), ("threads_per_lane", 100)])
    def test_rejects(self, field, value):
        with pytest.raises(lb.UsageError):
            lb.DecodeConfig(**{field: value}).validate()

    def test_cutoff(self):
        assert lb.compute_cutoff(2.0, 14.0) == 16.0
        with pytest.raises(lb.UsageError):
            lb.compute_cutoff(1.0, 0.0)


class TestGenerators:
    def test_hclg_shape(self):
        w = synthetic.hclg_graph(0, num_states=100_000, pool_size=2000)
        eps = w.arc_ilabel == 0
        L = 5
        assert np.all(w.arc_dst[eps] % L > w.arc_src[eps] % L)        # acyclic epsilon levels
        assert 2.5 < w.num_arcs / w.num_states < 3.6
        assert np.isfinite(w.final_cost_array).sum() > 0.005 * w.num_states
        assert np.all(np.diff(w.arc_offsets) >= 1)

    def test_c5_hubs(self):
        w = synthetic.hclg_graph(0, num_states=200_000, pool_size=4000, eps_depth=8, num_hubs=50,
                                 hub_share=0.3, eps_per_state=0.45)
        eps = w.arc_ilabel == 0
        indeg = np.bincount(w.arc_dst[eps], minlength=w.num_states)
        assert indeg.max() > 200
        assert np.all(w.arc_dst[eps] % 9 > w.arc_src[eps] % 9)

    def test_deterministic(self):
        a = synthetic.hclg_graph(4, num_states=20_000, pool_size=500)
        b = synthetic.hclg_graph(4, num_states=20_000, pool_size=500)
        assert np.array_equal(a.arc_dst, b.arc_dst) and np.array_equal(a.arc_weight, b.arc_weight)


class TestOracleKATs:
    """The reference's hand-sized vectors (conftest.py:8-28, test_decoder.py) on the oracle."""

    def test_w1(self, oracle_mod):
        r = oracle_mod.decode(lb.load_wfst_text(W1), lb.load_cost_matrix("1 2\n0.3 0.1\n"), 14.0, 8.0)
        assert r.words == [1] and r.alignment == [(1, 0)] and r.total_cost == pytest.approx(0.8)
        assert r.cutoffs.tolist() == pytest.approx([14.0, 14.8])
        assert len(r.final["from_"]) == 2

    def test_diamond(self, oracle_mod):
        w, m = lb.load_wfst_text(DIAMOND), lb.load_cost_matrix("3 2\n0.1 0.2\n0.1 0.2\n0.2 0.2\n")
        r = oracle_mod.decode(w, m, 14.0, 8.0)
        assert r.total_cost == pytest.approx(1.0)
        ex = sorted(np.round(np.concatenate([b[4] for b in r.blocks]), 9).tolist())
        assert ex == pytest.approx([0.0, 0.0, 0.0, 0.4, 0.4, 0.4])
        assert len(oracle_mod.decode(w, m, 14.0, 0.39).final["from_"]) == 3
        assert len(oracle_mod.decode(w, m, 14.0, 0.41).final["from_"]) == 6

    def test_failure_and_partial(self, oracle_mod):
        w = lb.load_wfst_text(W1)
        assert oracle_mod.decode(w, lb.load_cost_matrix("2 2\n0.3 0.1\n0.3 0.1\n"), 14.0).status == 1
        r = oracle_mod.decode(lb.load_wfst_text("0 1 1 1 0.5\n2 0.0\n"), lb.load_cost_matrix("1 1\n0.3\n"), 14.0)
        assert r.partial and r.words == [1]

    def test_eps_outputs(self, oracle_mod):
        w = lb.load_wfst_text("0 1 1 1 0.1\n1 2 1 0 0.1\n2 3 1 2 0.1\n3 0.0\n")
        r = oracle_mod.decode(w, lb.load_cost_matrix("3 1\n0.2\n0.2\n0.2\n"), 14.0)
        assert r.words == [1, 2] and r.total_cost == pytest.approx(0.9)

    def test_eps_closure_single_op(self, oracle_mod):
        w = lb.load_wfst_text("0 1 0 0 0.3\n1 2 0 0 0.4\n2 0.0\n")
        s, c = oracle_mod.expand_nonemitting(w, [0], [0.5], 100.0)
        assert s.tolist() == [0, 1, 2] and c == pytest.approx([0.5, 0.8, 1.2])

    def test_backtrace_cycle_is_bounded(self, oracle_mod):
        """the reference hangs here; the oracle must not."""
        w = lb.load_wfst_text("3 1 1 1 1.0\n3 2 1 2 1.0000000000009095\n1 2 0 0 0.0\n2 1 0 0 0.0\n1 0.0\n2 0.0\n")
        r = oracle_mod.decode(w, lb.load_cost_matrix("1 1\n0.0\n"), 10.0, want_lattice=False)
        assert r.status == 4 and "backtrace" in r.message

    def test_max_active_binds_and_counters(self, oracle_mod):
        g = synthetic.uniform_bench_graph(0, num_states=3000, arcs_per_state=5, num_labels=100)
        m = synthetic.bench_matrix(1, num_frames=20, num_labels=100)
        free = oracle_mod.decode(g, m, 13.0, want_lattice=False)
        capped = oracle_mod.decode(g, m, 13.0, max_active=200, want_lattice=False)
        assert max(len(f[0]) for f in free.frames) > 1000
        assert max(len(f[0]) for f in capped.frames[1:]) < 600
        assert capped.counters["n_cand"] < free.counters["n_cand"]
        assert free.counters["n_scan"] == 5 * free.counters["n_tokens"]
