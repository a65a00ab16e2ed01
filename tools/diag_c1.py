"""Diagnose a device/oracle divergence on C1 frames (first differing frame)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1804_03243_b200 as lb
from paper_1804_03243_b200 import synthetic
from oracle import oracle as O
w = synthetic.config_graph("C1")
for lat in (False, True):
    m = synthetic.bench_matrix(100, num_frames=20, num_labels=500)
    ref = O.decode(w, m, 13.0, lattice_beam=8.0, want_lattice=lat)
    got = lb.decode_utterance(w, m, lb.DecodeConfig(beam=13.0, lattice_beam=8.0, max_lattice_arcs=50_000_000),
                              want_lattice=lat, collect_frame_packs=True)
    print("lat", lat, "cost", got.total_cost, ref.total_cost)
    for f, ((s1, p1), (s2, p2)) in enumerate(zip(got.frame_packs, ref.frame_packs)):
        if not (np.array_equal(s1, s2) and np.array_equal(p1, p2)):
            a, b = set(s1.tolist()), set(s2.tolist())
            print(" frame", f, "n", len(s1), len(s2), "extra", sorted(a - b)[:5], "missing", sorted(b - a)[:5])
            common = np.intersect1d(s1, s2)
            i1 = np.searchsorted(s1, common); i2 = np.searchsorted(s2, common)
            bad = np.flatnonzero(p1[i1] != p2[i2])
            print("  pack mismatches", len(bad), [(int(common[k]), hex(int(p1[i1[k]])), hex(int(p2[i2[k]]))) for k in bad[:3]])
            cf = got.work_lattice.frames[f] if got.work_lattice else None
            break
