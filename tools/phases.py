"""Per-phase time breakdown of the decode kernel (LB_PHASE_PROFILE=1)."""
import os
import sys
import time

os.environ["LB_PHASE_PROFILE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1804_03243_b200 as lb
from paper_1804_03243_b200 import synthetic
from paper_1804_03243_b200.resident import decode_batch_resident

U = int(sys.argv[1]) if len(sys.argv) > 1 else 64
T = int(sys.argv[2]) if len(sys.argv) > 2 else 100
confs = [tuple(int(x) for x in a.split("x")) for a in (sys.argv[3:] or ["2x1024"])]
g = synthetic.hclg_graph(0)
mats = [torch.from_numpy(np.ascontiguousarray(synthetic.hclg_matrix(100 + i, num_frames=T).costs)).cuda()
        for i in range(U)]
for ctas, thr in confs:
    cfg = lb.DecodeConfig(beam=13.0, max_active=7000, ctas_per_lane=ctas, threads_per_lane=thr)
    decode_batch_resident(g, mats, cfg)
    outs, tm = decode_batch_resident(g, mats, cfg)
    lanes = min(U, 148 // ctas)
    per = {k: v / U / T * 1e3 for k, v in tm["phases_ms"].items()}
    print(f"ctas={ctas} thr={thr} kernel={tm['decode_ms']:.1f}ms  per-lane-frame us: " +
          " ".join(f"{k}={v:.1f}" for k, v in per.items()) + f"  total={sum(per.values()):.1f}")
