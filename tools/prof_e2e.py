import cProfile, pstats, os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1804_03243_b200 as lb
from paper_1804_03243_b200 import synthetic
g = synthetic.hclg_graph(0)
pool = [np.ascontiguousarray(synthetic.hclg_matrix(100 + i, num_frames=300).costs) for i in range(256)]
mats = [pool[i % 256] for i in range(4096)]
cfg = lb.DecodeConfig(beam=13.0, max_active=7000, lanes=64)
lb.decode_batch(g, mats, cfg, want_lattice=False)
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
lb.decode_batch(g, mats, cfg, want_lattice=False)
pr.disable()
print("wall", time.perf_counter() - t0)
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
