"""Golden vectors for lattice scoring, produced by the REFERENCE (run here only).

Lattices come from the CPU oracle's decodes of seeded random tasks and config-C1
frames (their FinalLattice arrays are stored, so the GPU box needs no decoder to
replay them); references are seeded random word sequences biased toward the
lattice's own words.  `latbeam.scoring` (/root/reference, read-only) computes
wer / oracle_wer / lattice_density.

    python tests/golden/make_scoring_golden.py      # writes tests/golden/scoring.npz
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from latbeam import lattice as RL  # noqa: E402
from latbeam import scoring as RS  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_1804_03243_b200 import synthetic  # noqa: E402


def main():
    out = {}
    k = 0
    rng = np.random.default_rng(20261017)
    tasks = [synthetic.random_task(s, allow_eps_cycles=False) for s in range(5000, 5060)]
    tasks += [synthetic.random_task(s, max_states=200, max_arcs=1200, num_labels=20, max_frames=30)
              for s in range(6000, 6010)]
    for w, m in tasks:
        res = O.decode(w, m, 9.0, lattice_beam=3.0)
        if not res.ok:
            continue
        f = res.final
        fl = RL.FinalLattice(int(f["num_nodes"]), int(f["start"]), f["final_ids"], f["final_costs"], f["from_"],
                             f["to"], f["ilabel"], f["olabel"], f["graph_cost"], f["acoustic_cost"],
                             f["node_frame"], f["node_idx"], int(f["num_frames"]))
        words = [int(x) for x in f["olabel"] if x > 0] or [1]
        nref = int(rng.integers(1, 8))
        ref = [int(words[rng.integers(len(words))]) if rng.random() < 0.7 else int(rng.integers(1, 40))
               for _ in range(nref)]
        try:
            ow = RS.oracle_wer(fl, ref)
        except Exception:   # noqa: BLE001 - no complete path
            ow = -1
        hyp = res.words
        wr = RS.wer(hyp, ref)
        for key in ("num_nodes", "start", "final_ids", "from_", "to", "ilabel", "olabel", "node_frame"):
            out[f"{k}/{key}"] = np.asarray(f[key])
        out[f"{k}/ref"] = np.asarray(ref, dtype=np.int64)
        out[f"{k}/hyp"] = np.asarray(hyp, dtype=np.int64)
        out[f"{k}/oracle_wer"] = np.int64(ow)
        out[f"{k}/wer"] = np.asarray([wr.substitutions, wr.insertions, wr.deletions], dtype=np.int64)
        out[f"{k}/density"] = np.float64(RS.lattice_density(fl))
        k += 1
    out["n"] = np.int64(k)
    np.savez_compressed(os.path.join(HERE, "scoring.npz"), **out)
    print("wrote", k, "cases")


if __name__ == "__main__":
    main()
