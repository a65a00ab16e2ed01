"""frames/s of every decode mode by batch size, on a config's graph (GPU box).

Checks the host's automatic mode choice (choose_mode in csrc/latbeam_b200.cu,
tuned on the C2 graph) on other graph shapes: forced batched mode, 2/3/4/8-CTA
lanes, and auto.  Costs HBM-resident; 1-best (C1 with lattices via the public API
when --lattice).
usage: python tools/mode_sweep.py C1|C2|C3|C5 [--lattice] [U ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1804_03243_b200 as lb
from paper_1804_03243_b200 import synthetic
from paper_1804_03243_b200.resident import decode_batch_resident

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
lattice = "--lattice" in sys.argv
Us = [int(x) for x in sys.argv[2:] if x != "--lattice"] or [1, 4, 8, 16, 32, 44, 64]
T = 150
g = synthetic.config_graph(name)
d = synthetic.CONFIGS[name]["decode"]
pool = [torch.from_numpy(np.ascontiguousarray(synthetic.config_matrix(name, u, num_frames=T).costs)).cuda()
        for u in range(16)]
modes = [("auto", None, 0), ("batched", "batched", 0), ("lane2", "lane", 2), ("lane3", "lane", 3),
         ("lane4", "lane", 4), ("lane8", "lane", 8), ("lane16", "lane", 16)]
for U in Us:
    tens = [pool[u % 16] for u in range(U)]
    row = []
    ref = None
    for label, mode, ctas in modes:
        if mode:
            os.environ["LB_MODE"] = mode
        else:
            os.environ.pop("LB_MODE", None)
        cfg = lb.DecodeConfig(beam=d["beam"], max_active=d["max_active"], ctas_per_lane=ctas,
                              lattice_beam=d["lattice_beam"], max_lattice_arcs=50_000_000)
        try:
            outs, _ = decode_batch_resident(g, tens, cfg, want_lattice=lattice)
            bad = [o["status"] for o in outs if o["status"] != 0]
            if bad:
                row.append(f"{label}=status{bad[0]}")
                continue
            costs = [o["total_cost"] for o in outs]
            ref = ref if label != "auto" else costs
            ms = min(decode_batch_resident(g, tens, cfg, want_lattice=lattice)[1]["decode_ms"] for _ in range(2))
            row.append(f"{label}={U * T / ms * 1e3 / 1e3:.1f}k" + ("" if costs == ref else "(MISMATCH)"))
        except Exception as exc:   # noqa: BLE001 - e.g. clusters that cannot be co-resident
            row.append(f"{label}=err({type(exc).__name__})")
    print(f"{name} U={U}: " + " ".join(row), flush=True)
