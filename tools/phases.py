"""Per-phase time breakdown of the decode kernel (LB_PHASE_PROFILE=1) and the
per-lane-frame work counters, on the bench workload (C2 graph, beam 13, max-active 7000).
usage: python tools/phases.py U T CxTHREADS [CxTHREADS ...]"""
import os
import sys

os.environ.setdefault("LB_PHASE_PROFILE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1804_03243_b200 as lb
from paper_1804_03243_b200 import synthetic
from paper_1804_03243_b200.resident import decode_batch_resident

U = int(sys.argv[1]) if len(sys.argv) > 1 else 64
T = int(sys.argv[2]) if len(sys.argv) > 2 else 100
confs = [tuple(int(x) for x in a.split("x")) for a in (sys.argv[3:] or ["2x768"])]
import json
g = synthetic.hclg_graph(0, **json.loads(os.environ.get("LB_GRAPH_KW", "{}")))
mats = [torch.from_numpy(np.array(synthetic.hclg_matrix(100 + i, num_frames=T).costs)).cuda()
        for i in range(U)]
names = ("tok", "scan", "cand", "efront", "escan", "ecand", "next", "lat")
for ctas, thr in confs:
    cfg = lb.DecodeConfig(beam=13.0, max_active=7000, ctas_per_lane=ctas, threads_per_lane=thr,
                          lanes=int(os.environ.get("LB_PHASE_LANES", U)))
    decode_batch_resident(g, mats, cfg)
    outs, tm = decode_batch_resident(g, mats, cfg)
    per = {k: v / U / T * 1e3 for k, v in tm["phases_ms"].items()}
    cnt = np.sum([o["counters"] for o in outs], axis=0) / (U * T)
    print(f"U={U} ctas={ctas} thr={thr} kernel={tm['decode_ms']:.1f}ms frames/s={U * T / tm['decode_ms'] * 1e3:.0f} "
          f"per-lane-frame us: " + " ".join(f"{k}={v:.1f}" for k, v in per.items()) +
          f" total={sum(per.values()):.1f}")
    print("   per lane-frame counts: " + " ".join(f"{n}={c:.0f}" for n, c in zip(names, cnt)), flush=True)
    wb, wn = tm["warp_busy_ms"], tm["warp_samples"]
    print("   avg warp busy us per occurrence: " + " ".join(
        f"{k}={wb[k] / wn[k] * 1e3:.1f}" for k in wb if wn[k] > 0), flush=True)
