"""One batched-mode decode of the bench workload at U lanes x T frames (for ncu launch lists)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1804_03243_b200 as lb
from paper_1804_03243_b200 import synthetic
from paper_1804_03243_b200.resident import decode_batch_resident

U = int(sys.argv[1]) if len(sys.argv) > 1 else 64
T = int(sys.argv[2]) if len(sys.argv) > 2 else 30
g = synthetic.hclg_graph(0)
mats = [torch.from_numpy(np.array(synthetic.hclg_matrix(100 + i, num_frames=T).costs)).cuda() for i in range(U)]
cfg = lb.DecodeConfig(beam=13.0, max_active=7000, lanes=U)
decode_batch_resident(g, mats, cfg)      # warm-up (workspace, graph capture)
ms = min(decode_batch_resident(g, mats, cfg)[1]["decode_ms"] for _ in range(3))
print(f"{ms:.2f} ms  {U * T / ms * 1e3:.0f} frames/s")
