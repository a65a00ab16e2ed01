"""Tiny lane-kernel decodes for compute-sanitizer racecheck (2-CTA lanes, 1-best and lattice)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_03243_b200 as lb
from paper_1804_03243_b200 import synthetic

os.environ["LB_MODE"] = "lane"
os.environ["LB_ZC_MIN"] = "1"   # progressive zero-copy staging even for 2 utterances
C = int(sys.argv[1]) if len(sys.argv) > 1 else 2
w = synthetic.hclg_graph(5, num_states=5000, pool_size=200, num_pdfs=50)
ms = [synthetic.hclg_matrix(9 + i, num_frames=3, num_pdfs=50) for i in range(2)]
q = lb.decode_batch(w, ms, lb.DecodeConfig(beam=8.0, max_active=100, ctas_per_lane=C), want_lattice=False)
r = lb.decode_batch(w, ms, lb.DecodeConfig(beam=8.0, lattice_beam=2.0, max_active=100, ctas_per_lane=C))
assert [x.total_cost for x in q] == [x.total_cost for x in r]
print("ok", C, [x.total_cost for x in q])
