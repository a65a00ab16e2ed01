"""Where the e2e (public API, host costs) time of the C4 job goes: the C-ABI call
(staging ring + decode + readback) vs the Python result assembly.
usage: python tools/e2e_split.py [utts]  (GPU box)"""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1804_03243_b200 as lb
from paper_1804_03243_b200 import _lib, synthetic
from paper_1804_03243_b200 import decoder as dec

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
g = synthetic.hclg_graph(0)
pool = [np.ascontiguousarray(synthetic.hclg_matrix(100 + i, num_frames=300).costs) for i in range(256)]
mats = [pool[i % 256] for i in range(n)]
cfg = lb.DecodeConfig(beam=13.0, max_active=7000, lanes=64)
lb.decode_batch(g, mats, cfg, want_lattice=False)
for rep in range(2):
    t0 = time.perf_counter()
    lb.decode_batch(g, mats, cfg, want_lattice=False)
    t_all = time.perf_counter() - t0
    L = _lib.lib()
    dg = dec.device_graph(g, 0)
    cptrs = (_lib.PD * n)(*[m.ctypes.data_as(_lib.PD) for m in mats])
    T = np.full(n, 300, dtype=np.int32)
    c = cfg.to_c(False, False)
    res = _lib.PV()
    t0 = time.perf_counter()
    rc = L.lb_decode_batch(dg.handle, n, cptrs, T.ctypes.data_as(_lib.P32), 3000, C.byref(c), C.byref(res))
    t_c = time.perf_counter() - t0
    t0 = time.perf_counter()
    out = dec.collect_results(g, res, mats, cfg, False, False, False, time.perf_counter())
    t_py = time.perf_counter() - t0
    tm = dec.result_timing(res)
    L.lb_result_free(res)
    print(f"n={n} decode_batch {t_all:.3f}s = C call {t_c:.3f}s (decode {tm['decode_ms']:.0f} ms, "
          f"h2d/stage {tm['h2d_ms']:.0f} ms, d2h {tm['d2h_ms']:.0f} ms) + python results {t_py:.3f}s; "
          f"frames/s public {n * 300 / t_all:.0f}, C {n * 300 / t_c:.0f}", flush=True)
