"""Seeded workloads: the reference's generators (restated) and an HCLG-like graph.

* `random_wfst` / `random_matrix` / `random_task` / `uniform_bench_graph` /
  `skewed_bench_graph` / `bench_matrix` draw exactly the same numpy
  `default_rng` sequence as the reference generators (synthetic.py:19-137 of
  `latbeam`), so seeds name the same graphs and matrices; tests/golden pins this
  by hashing the generated arrays against the reference's own output.
* `hclg_graph` is this package's generator for configs C2/C3/C4/C5
  (SURVEY.md §8(d)): a decoding-graph-shaped WFST with a per-state self-loop on
  the state's pdf, forward emitting arcs, a reconvergent high-out-degree "hot
  pool" (so max-active binds every frame), acyclic forward epsilon arcs of
  bounded chain depth, optional epsilon hub states (C5 back-off fan-in), ~10 %
  word-bearing arcs and ~1 % final states.  It assembles the CSR directly in
  state order (no text, no global sort) so 50M-arc graphs build in seconds.
"""

from __future__ import annotations

import numpy as np

from .acoustics import CostMatrix
from .wfst import Wfst, from_arcs


# ---------------------------------------------------------------------------
# Reference generators (same RNG draw order as synthetic.py:19-137)
# ---------------------------------------------------------------------------

def _emit_arc(rng, s, n, num_labels, num_words):
    d = int(rng.integers(0, n))
    il = int(rng.integers(1, num_labels + 1))
    ol = int(rng.integers(0, num_words + 1))
    w = float(rng.uniform(0.0, 3.0))
    return s, d, il, ol, w


def random_wfst(rng: np.random.Generator, max_states: int = 50, max_arcs: int = 200,
                num_labels: int = 8, num_words: int = 20, eps_prob: float = 0.2,
                allow_eps_cycles: bool = False, final_prob: float = 0.6) -> Wfst:
    """Random decodable graph; every state owns >= 1 emitting arc, state 0 starts."""
    n = int(rng.integers(2, max_states + 1))
    arcs = [_emit_arc(rng, s, n, num_labels, num_words) for s in range(n)]
    extra = int(rng.integers(0, max(max_arcs - n, 0) + 1))
    for _ in range(extra):
        s = int(rng.integers(0, n))
        if rng.random() < eps_prob and (allow_eps_cycles or s < n - 1):
            d = int(rng.integers(0, n)) if allow_eps_cycles else int(rng.integers(s + 1, n))
            ol = int(rng.integers(0, num_words + 1))
            w = float(rng.uniform(0.0, 3.0))
            arcs.append((s, d, 0, ol, w))
        else:
            arcs.append(_emit_arc(rng, s, n, num_labels, num_words))
    finals = [s for s in range(n) if rng.random() < final_prob] or [n - 1]
    fc = {s: float(rng.uniform(0.0, 2.0)) for s in finals}
    cols = list(zip(*arcs))
    return from_arcs(n, 0, np.asarray(cols[0], dtype=np.int32), np.asarray(cols[1], dtype=np.int32),
                     np.asarray(cols[2], dtype=np.int32), np.asarray(cols[3], dtype=np.int32),
                     np.asarray(cols[4], dtype=np.float64), fc)


def random_matrix(rng: np.random.Generator, num_labels: int, max_frames: int = 20,
                  allow_negative: bool = False) -> CostMatrix:
    t = int(rng.integers(1, max_frames + 1))
    return CostMatrix(rng.uniform(-1.0 if allow_negative else 0.0, 5.0, size=(t, num_labels)))


def random_task(seed: int, max_states: int = 50, max_arcs: int = 200, num_labels: int = 8,
                max_frames: int = 20, allow_eps_cycles: bool = False,
                allow_negative: bool = False) -> tuple[Wfst, CostMatrix]:
    rng = np.random.default_rng(seed)
    w = random_wfst(rng, max_states=max_states, max_arcs=max_arcs, num_labels=num_labels,
                    allow_eps_cycles=allow_eps_cycles)
    return w, random_matrix(rng, num_labels, max_frames=max_frames, allow_negative=allow_negative)


def _csr(num_states, src, dst, il, ol, wt, finals) -> Wfst:
    return from_arcs(num_states, 0, src, dst.astype(np.int32), il.astype(np.int32),
                     ol.astype(np.int32), wt, finals)


def uniform_bench_graph(seed: int, num_states: int = 5000, arcs_per_state: int = 24,
                        num_labels: int = 32) -> Wfst:
    """Same out-degree everywhere (config C1 uses 10000 x 5, 500 labels)."""
    rng = np.random.default_rng(seed)
    total = num_states * arcs_per_state
    src = np.repeat(np.arange(num_states, dtype=np.int64), arcs_per_state)
    dst = rng.integers(0, num_states, size=total, dtype=np.int64)
    il = rng.integers(1, num_labels + 1, size=total, dtype=np.int64)
    ol = rng.integers(0, num_labels + 1, size=total, dtype=np.int64)
    wt = rng.uniform(0.0, 3.0, size=total)
    return _csr(num_states, src, dst, il, ol, wt, np.zeros(num_states))


def skewed_bench_graph(seed: int, num_states: int = 5000, arcs_per_state: int = 24,
                       num_labels: int = 32, hub_share: float = 0.3) -> Wfst:
    """One hub state owns `hub_share` of all arcs."""
    rng = np.random.default_rng(seed)
    total = num_states * arcs_per_state
    hub = int(total * hub_share)
    per_other = max((total - hub) // (num_states - 1), 1)
    src = np.concatenate([np.zeros(hub, dtype=np.int64),
                          np.repeat(np.arange(1, num_states, dtype=np.int64), per_other)])
    n = len(src)
    dst = rng.integers(0, num_states, size=n, dtype=np.int64)
    il = rng.integers(1, num_labels + 1, size=n, dtype=np.int64)
    ol = rng.integers(0, num_labels + 1, size=n, dtype=np.int64)
    wt = rng.uniform(0.0, 3.0, size=n)
    return _csr(num_states, src, dst, il, ol, wt, np.zeros(num_states))


def bench_matrix(seed: int, num_frames: int = 500, num_labels: int = 32) -> CostMatrix:
    rng = np.random.default_rng(seed)
    return CostMatrix(rng.uniform(0.0, 5.0, size=(num_frames, num_labels)))


# ---------------------------------------------------------------------------
# HCLG-like generator (configs C2-C5)
# ---------------------------------------------------------------------------

def hclg_graph(seed: int = 0, num_states: int = 5_000_000, num_pdfs: int = 3000,
               pool_size: int = 30_000, pool_fwd: int = 6, pool_share: float = 0.9,
               cold_fwd_mean: float = 1.6, cold_to_pool: float = 0.5,
               eps_per_state: float = 0.4, eps_depth: int = 4, eps_to_pool: float = 0.7,
               num_hubs: int = 0, hub_share: float = 0.0, word_share: float = 0.1,
               num_words: int = 30_000, final_share: float = 0.01) -> Wfst:
    """Decoding-graph-shaped WFST, assembled directly in CSR order.

    Per state s (in arc-id order): a self-loop labelled pdf(s); forward
    emitting arcs s->d labelled pdf(d) (pool states: `pool_fwd` arcs, a share
    `pool_share` landing in the pool; cold states: 1 + Poisson-ish extra with
    mean `cold_fwd_mean`, a share `cold_to_pool` landing in the pool); then
    epsilon arcs.  Epsilon arcs only climb `level(s) = s % (eps_depth+1)`, so
    epsilon chains are acyclic with depth <= eps_depth.
    With `num_hubs` > 0, a share `hub_share` of epsilon arcs targets the hub
    states (ids at the top level), giving each an in-degree of
    ~hub_share*eps/num_hubs.  Weights U(0,3); finals U(0,2).
    """
    rng = np.random.default_rng(seed)
    S = int(num_states)
    P = min(int(pool_size), S)
    L = eps_depth + 1
    pdf = rng.integers(1, num_pdfs + 1, size=S, dtype=np.int64)

    n_fwd = np.empty(S, dtype=np.int64)
    n_fwd[:P] = pool_fwd
    extra = rng.random(S - P) < (cold_fwd_mean - 1.0) if cold_fwd_mean < 2 else None
    if extra is not None:
        n_fwd[P:] = 1 + extra
    else:
        n_fwd[P:] = 1 + rng.poisson(cold_fwd_mean - 1.0, size=S - P)
    n_eps = (rng.random(S) < eps_per_state).astype(np.int64)
    level = np.arange(S, dtype=np.int64) % L
    n_eps[level == L - 1] = 0          # top level has nowhere higher to go
    deg = 1 + n_fwd + n_eps
    off = np.zeros(S + 1, dtype=np.int64)
    np.cumsum(deg, out=off[1:])
    A = int(off[-1])

    src = np.repeat(np.arange(S, dtype=np.int64), deg)
    # position of each arc within its state: 0 = self-loop, 1..n_fwd = forward, rest = eps
    k = np.arange(A, dtype=np.int64) - np.repeat(off[:-1], deg)
    nf_rep = np.repeat(n_fwd, deg)
    is_self = k == 0
    is_fwd = (k >= 1) & (k <= nf_rep)
    is_eps = k > nf_rep

    dst = np.empty(A, dtype=np.int64)
    dst[is_self] = src[is_self]
    fsrc = src[is_fwd]
    to_pool = np.where(fsrc < P, rng.random(len(fsrc)) < pool_share,
                       rng.random(len(fsrc)) < cold_to_pool)
    fdst = np.where(to_pool, rng.integers(0, P, size=len(fsrc)), rng.integers(0, S, size=len(fsrc)))
    dst[is_fwd] = fdst

    esrc = src[is_eps]
    ne = len(esrc)
    # pick a destination with strictly higher level: d = base*L + lvl', lvl' in (level(s), L-1]
    elev = esrc % L
    up = elev + 1 + (rng.random(ne) * (L - 1 - elev)).astype(np.int64)
    up = np.minimum(up, L - 1)
    in_pool = rng.random(ne) < eps_to_pool
    span = np.where(in_pool, max(P // L, 1), max((S - L) // L + 1, 1))
    base = (rng.random(ne) * span).astype(np.int64)
    edst = np.minimum(base * L + up, S - 1)
    if num_hubs > 0 and hub_share > 0:
        hubs = (np.arange(num_hubs, dtype=np.int64) * ((S - L) // L // num_hubs)) * L + (L - 1)
        hub_pick = rng.random(ne) < hub_share
        edst = np.where(hub_pick, hubs[rng.integers(0, num_hubs, size=ne)], edst)
    assert np.all(edst % L > elev), "epsilon arcs must climb levels (acyclic)"
    dst[is_eps] = edst

    il = np.zeros(A, dtype=np.int64)
    il[is_self] = pdf[src[is_self]]
    il[is_fwd] = pdf[fdst]
    ol = np.zeros(A, dtype=np.int64)
    words = rng.random(A) < word_share
    words &= ~is_self
    ol[words] = rng.integers(1, num_words + 1, size=int(words.sum()))
    wt = rng.uniform(0.0, 3.0, size=A)

    final = np.full(S, np.inf)
    fin = rng.random(S) < final_share
    fin[:P:97] = True
    final[fin] = rng.uniform(0.0, 2.0, size=int(fin.sum()))
    return Wfst(S, 0, off, src.astype(np.int32), dst.astype(np.int32), il.astype(np.int32),
                ol.astype(np.int32), wt, final)


def hclg_matrix(seed: int, num_frames: int = 300, num_pdfs: int = 3000) -> CostMatrix:
    """i.i.d. U(0,5) f64 acoustic costs."""
    rng = np.random.default_rng(seed)
    return CostMatrix(rng.uniform(0.0, 5.0, size=(num_frames, num_pdfs)))


CONFIGS = {
    # name: (graph kwargs, decode kwargs, frames, utterances)
    "C1": dict(graph=("uniform", dict(seed=0, num_states=10_000, arcs_per_state=5, num_labels=500)),
               decode=dict(beam=13.0, lattice_beam=8.0, max_active=0), frames=300, utts=20,
               want_lattice=True),
    "C2": dict(graph=("hclg", dict(seed=0)), decode=dict(beam=13.0, lattice_beam=8.0, max_active=7000),
               frames=300, utts=1, want_lattice=False),
    "C3": dict(graph=("hclg", dict(seed=0)), decode=dict(beam=13.0, lattice_beam=8.0, max_active=7000),
               frames=300, utts=1, want_lattice=True),
    "C4": dict(graph=("hclg", dict(seed=0)), decode=dict(beam=13.0, lattice_beam=8.0, max_active=7000),
               frames=300, utts=4096, want_lattice=False),
    # ~1000 backoff hubs with epsilon in-degree ~8.5k each (most states carry an
    # epsilon "backoff" arc into a hub, as an LM graph does)
    "C5": dict(graph=("hclg", dict(seed=0, num_states=15_000_000, pool_size=60_000, pool_fwd=8,
                                   cold_fwd_mean=1.6, eps_per_state=0.8, eps_depth=8,
                                   num_hubs=1000, hub_share=0.8)),
               decode=dict(beam=16.0, lattice_beam=8.0, max_active=20_000), frames=300, utts=1,
               want_lattice=False),
}


def config_graph(name: str) -> Wfst:
    kind, kw = CONFIGS[name]["graph"]
    return uniform_bench_graph(**kw) if kind == "uniform" else hclg_graph(**kw)


def config_matrix(name: str, utt: int, num_frames: int | None = None) -> CostMatrix:
    c = CONFIGS[name]
    t = num_frames or c["frames"]
    if name == "C1":
        return bench_matrix(100 + utt, num_frames=t, num_labels=500)
    return hclg_matrix(100 + utt, num_frames=t, num_pdfs=3000)
