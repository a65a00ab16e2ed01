"""Time the REAL reference decoder (`latbeam`, installed into baseline/_ref by
`pip install --target baseline/_ref`) on config C1, on this host's CPU cores:

  (i)  the reference's own decode_batch(num_workers=ncores) (a thread pool over
       utterances, decoder.py:644-672);
  (ii) ncores processes x decode_utterance(num_workers=1) (the best-case CPU
       figure);

both with the numba engine (and (ii) also with the numpy engine), 1-best +
lattice as C1 specifies, on a bounded sample: ncores utterances x the first
`--frames` frames of C1's matrices.  Prints one JSON line.  A measurement aid
(no part of the product path); run it on the GPU box:

    python tools/reference_c1.py [--frames 60] > profiles/r02_reference_c1.json
"""

from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


def _setup(numba: bool):
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_ref")
    os.environ["LATBEAM_NUMBA"] = "1" if numba else "0"
    sys.path.insert(0, REF)
    import latbeam
    latbeam.use_numba(numba)
    return latbeam


def _inputs(latbeam, n, frames):
    from latbeam import synthetic as RS
    w = RS.uniform_bench_graph(0, num_states=10_000, arcs_per_state=5, num_labels=500)
    mats = [latbeam.CostMatrix(RS.bench_matrix(100 + i, num_frames=300, num_labels=500).costs[:frames].copy())
            for i in range(n)]
    return w, mats


def _one(args):
    i, frames, numba = args
    latbeam = _setup(numba)
    w, mats = _inputs(latbeam, i + 1, frames)
    cfg = latbeam.DecodeConfig(beam=13.0, lattice_beam=8.0, max_lattice_arcs=20_000_000, num_workers=1)
    latbeam.decode_utterance(w, latbeam.CostMatrix(mats[i].costs[:2].copy()), cfg)   # JIT / page-in
    t0 = time.perf_counter()
    r = latbeam.decode_utterance(w, mats[i], cfg)
    return time.perf_counter() - t0, r.total_cost


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=60)
    ap.add_argument("--procs", type=int, default=0)
    a = ap.parse_args()
    if not os.path.isdir(os.path.join(REF, "latbeam")):
        print(json.dumps({"unavailable": "baseline/_ref has no latbeam install"}))
        return
    n = a.procs or len(os.sched_getaffinity(0))
    out = {"config": "C1: uniform_bench_graph(0, 10000, 5, 500), beam 13, lattice beam 8, 1-best + lattice",
           "sample": f"{n} utterances x first {a.frames} frames", "cores": n}
    # (ii) ncores processes x decode_utterance(num_workers=1)
    ctx = mp.get_context("spawn")
    for numba in (True, False):
        with ctx.Pool(n) as pool:
            pool.map(_one, [(0, 2, numba)] * n)            # compile caches / imports in every worker
            t0 = time.perf_counter()
            res = pool.map(_one, [(i, a.frames, numba) for i in range(n)])
            wall = time.perf_counter() - t0
        key = "processes_numba" if numba else "processes_numpy"
        out[key] = {"frames_per_s": n * a.frames / wall, "wall_s": wall,
                    "per_utt_s_median": sorted(r[0] for r in res)[n // 2]}
    # (i) decode_batch(num_workers=ncores), numba engine, one process
    latbeam = _setup(True)
    w, mats = _inputs(latbeam, n, a.frames)
    cfg = latbeam.DecodeConfig(beam=13.0, lattice_beam=8.0, max_lattice_arcs=20_000_000, num_workers=n)
    latbeam.decode_batch(w, [latbeam.CostMatrix(m.costs[:2].copy()) for m in mats[:2]], cfg)
    t0 = time.perf_counter()
    latbeam.decode_batch(w, mats, cfg)
    wall = time.perf_counter() - t0
    out["decode_batch_numba"] = {"frames_per_s": n * a.frames / wall, "wall_s": wall}
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                out["cpu"] = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
