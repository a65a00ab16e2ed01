"""Where does a lattice decode spend its time?  C1 (20 utts) and C3 (1 utt)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1804_03243_b200 as lb
from paper_1804_03243_b200 import synthetic

for name, n in (("C1", int(sys.argv[1]) if len(sys.argv) > 1 else 4), ("C3", 1)):
    g = synthetic.config_graph(name)
    d = synthetic.CONFIGS[name]["decode"]
    mats = [np.ascontiguousarray(synthetic.config_matrix(name, u).costs) for u in range(n)]
    cfg = lb.DecodeConfig(beam=d["beam"], lattice_beam=d["lattice_beam"], max_active=d["max_active"],
                          max_lattice_arcs=50_000_000)
    lb.decode_batch(g, mats, cfg)
    for rep in range(int(os.environ.get("REPS", "3"))):
      t0 = time.perf_counter()
      res = lb.decode_batch(g, mats, cfg, collect_timings=True)
      wall = time.perf_counter() - t0
      tm = res[0].timings
      print(f"{name} x{n}: wall {wall:.2f}s  decode {tm['token_passing']:.3f}s prune {tm['lattice_pruning']:.3f}s "
            f"h2d {tm['h2d']:.3f}s d2h {tm['d2h']:.3f}s  host-rest {wall - tm['token_passing'] - tm['lattice_pruning'] - tm['h2d'] - tm['d2h']:.2f}s  "
            f"live arcs/utt {np.mean([r.counters['n_lat'] for r in res]):.0f} final arcs/utt {np.mean([r.lattice.num_arcs for r in res]):.0f}",
            flush=True)
