"""Single-utterance public-API timing (C2 / C5 graphs): wall vs library decode / h2d, per
staging / mode variant (environment knobs of csrc/latbeam_b200.cu)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1804_03243_b200 as lb
from paper_1804_03243_b200 import synthetic

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
g = synthetic.config_graph(name)
d = synthetic.CONFIGS[name]["decode"]
m = [np.ascontiguousarray(synthetic.config_matrix(name, 0).costs)]
cfg = lb.DecodeConfig(beam=d["beam"], max_active=d["max_active"])
VARIANTS = {"auto": {}, "batched": {"LB_MODE": "batched"}, "copy": {"LB_E2E_COPY": "1"},
            "noprog": {"LB_NO_PROGRESSIVE": "1"}}
for mode in ("auto", "batched", "copy", "noprog", "auto"):
    for k in ("LB_MODE", "LB_E2E_COPY", "LB_NO_PROGRESSIVE"):
        os.environ.pop(k, None)
    os.environ.update(VARIANTS[mode])
    lb.decode_batch(g, m, cfg, want_lattice=False)
    for _ in range(3):
        t0 = time.perf_counter()
        r = lb.decode_batch(g, m, cfg, want_lattice=False, collect_timings=True)
        wall = (time.perf_counter() - t0) * 1e3
        tm = r[0].timings
        print(f"{name} {mode:8s} wall {wall:6.2f} ms  decode {tm['token_passing'] * 1e3:6.2f}  h2d {tm['h2d'] * 1e3:5.2f}  "
              f"d2h {tm['d2h'] * 1e3:5.2f}", flush=True)
