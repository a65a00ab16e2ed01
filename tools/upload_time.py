"""Graph ingestion timing: C5 generation, device replica build (lb_graph_create), npz I/O."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_03243_b200 as lb
from paper_1804_03243_b200 import synthetic

lb.device_graph(synthetic.uniform_bench_graph(0, num_states=100, arcs_per_state=2, num_labels=4), 0)  # CUDA init
t0 = time.perf_counter()
w = synthetic.config_graph("C5")
t1 = time.perf_counter()
g = lb.device_graph(w, 0)
t2 = time.perf_counter()
print(f"C5 ({w.num_arcs / 1e6:.1f}M arcs) generate {t1 - t0:.2f}s  device replica (lb_graph_create) {t2 - t1:.3f}s  "
      f"{g.device_bytes / 1e9:.2f} GB")
p = "/tmp/c5.npz"
t3 = time.perf_counter()
lb.save_wfst_npz(w, p)
t4 = time.perf_counter()
lb.load_wfst_npz(p)
t5 = time.perf_counter()
print(f"npz save {t4 - t3:.2f}s load {t5 - t4:.2f}s")
