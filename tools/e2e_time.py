"""e2e timing of decode_batch on the C4 workload (64 x 300 frames, host numpy costs)
under the staging variants: progressive zero-copy (default), LB_NO_PROGRESSIVE=1,
LB_E2E_COPY=1.  Prints wall ms per call and the library's decode / h2d timings."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1804_03243_b200 as lb
from paper_1804_03243_b200 import synthetic

U = int(sys.argv[1]) if len(sys.argv) > 1 else 64
T = 300
g = synthetic.hclg_graph(0)
mats = [np.ascontiguousarray(synthetic.hclg_matrix(100 + i, num_frames=T).costs) for i in range(2 * U)]
cfg = lb.DecodeConfig(beam=13.0, max_active=7000)
print("cpus", os.cpu_count(), flush=True)
VARIANTS = {"progressive": {}, "no_progressive": {"LB_NO_PROGRESSIVE": "1"}, "copy": {"LB_E2E_COPY": "1"},
            "st2": {"LB_STAGE_THREADS": "2"}, "st4": {"LB_STAGE_THREADS": "4"}, "st8": {"LB_STAGE_THREADS": "8"}}
names = sys.argv[2].split(",") if len(sys.argv) > 2 else ["progressive", "no_progressive", "copy"]
for name in names:
    env = VARIANTS[name]
    for k, v in env.items():
        os.environ[k] = v
    lb.decode_batch(g, mats[:U], cfg, want_lattice=False)
    walls, dec, h2d = [], [], []
    for rep in range(4):
        m = mats[U * (rep % 2):U * (rep % 2) + U]
        t0 = time.perf_counter()
        res = lb.decode_batch(g, m, cfg, want_lattice=False, collect_timings=True)
        walls.append((time.perf_counter() - t0) * 1e3)
        dec.append(res[0].timings["token_passing"] * 1e3)
        h2d.append(res[0].timings["h2d"] * 1e3)
    print(f"{name:15s} wall ms {np.median(walls):7.1f} (min {min(walls):.1f})  decode {np.median(dec):6.1f}  "
          f"h2d/stage {np.median(h2d):6.1f}  -> {U * T / np.median(walls) * 1e3:,.0f} frames/s", flush=True)
    for k in env:
        del os.environ[k]
