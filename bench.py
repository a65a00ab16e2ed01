"""Benchmark: decoded frames/s (and arcs/s) of the B200 decoder on config C4.

Workload (BASELINE.json configs[3], "sequence-parallel batch"): the C2/C3
HCLG-shaped graph (5M states, ~14.7M arcs, 3000 pdfs, acyclic epsilons),
beam 13, max-active 7000, 1-best, T=300-frame utterances of i.i.d. U(0,5) f64
acoustic costs.  One step = one batch of `--utts` utterances decoded to the
end on every GPU (one decode lane per utterance; weak scaling over ranks).

  value  frames/s with the cost matrices already resident in HBM (C-ABI
         lb_decode_batch_device, CUDA events on the launching stream, L2
         flushed between steps), max over ranks, whole box.
  e2e    the same metric through the public API `decode_batch` on host numpy
         matrices: H2D of the costs and D2H of the results inside the timed region.

`--impl reference` times the reference algorithm's CPU path instead (the
oracle/ C port of latbeam's decoder, all host threads), on a bounded sample.

    python bench.py [--gpus N --steps K --warmup W]
    torchrun --nproc-per-node N bench.py --gpus N ...
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decoded frames/sec & arcs/sec (whole box) at 1/2/4/8 B200 vs CPU reference"
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
PROFILE_SUMMARY = os.path.join(ROOT, "profiles", "decode_kernel_traffic.json")


def bytes_of(c):
    """Algorithmic bytes of a decode, from the device counters
    [tokens, arcs scanned, candidates, eps frontier, eps arcs, eps candidates,
    tokens kept, lattice arcs]."""
    return (28 * c[0] + 16 * c[1] + 8 * c[2] + 28 * c[3] + 16 * c[4] + 8 * c[5] + 24 * c[6]
            + 16 * c[7])


def parse_args(argv=None):
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--utts", type=int, default=int(os.environ.get("LB_BENCH_UTTS", 64)),
                   help="utterances per step per GPU (= decode lanes)")
    p.add_argument("--frames", type=int, default=300)
    p.add_argument("--lanes", type=int, default=0)
    p.add_argument("--threads", type=int, default=0, help="threads per CTA of a lane")
    p.add_argument("--ctas", type=int, default=0, help="CTAs (thread-block cluster size) per lane")
    p.add_argument("--states", type=int, default=5_000_000)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--cpu-utts", type=int, default=0)
    p.add_argument("--cpu-frames", type=int, default=100)
    p.add_argument("--no-configs", action="store_true", help="skip the C1/C2/C3 side measurements")
    p.add_argument("--all-configs", action="store_true", help="also measure C5 (builds the 50M-arc graph)")
    return p.parse_args(argv)


class Dist:
    def __init__(self, backend_gpu=True):
        self.rank = int(os.environ.get("RANK", 0))
        self.world = int(os.environ.get("WORLD_SIZE", 1))
        self.local = int(os.environ.get("LOCAL_RANK", 0))
        self.pg = None
        if self.world > 1:
            import torch.distributed as dist
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            backend = "nccl" if backend_gpu else "gloo"
            if backend_gpu:
                import torch
                torch.cuda.set_device(self.local)
            dist.init_process_group(backend)
            self.pg = dist

    def max(self, x: float) -> float:
        if self.pg is None:
            return x
        import torch
        dev = f"cuda:{self.local}" if self.pg.get_backend() == "nccl" else "cpu"
        t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def sum(self, x: float) -> float:
        if self.pg is None:
            return x
        import torch
        dev = f"cuda:{self.local}" if self.pg.get_backend() == "nccl" else "cpu"
        t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
        self.pg.all_reduce(t)
        return float(t.item())

    def barrier(self):
        if self.pg is not None:
            self.pg.barrier()

    def close(self):
        if self.pg is not None:
            self.pg.destroy_process_group()


def shard_seeds(rank: int, step: int, utts: int, pool: int) -> list[int]:
    """Utterance seeds of one rank's step: disjoint across ranks (rank-major),
    cycling through a pool of `pool` distinct utterances per rank."""
    base = 100 + rank * 1_000_000
    return [base + (step * utts + i) % pool for i in range(utts)]


class ClockSampler:
    """nvidia-smi clock / throttle sampling during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.th = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.th = threading.Thread(target=self._read, daemon=True)
        self.th.start()

    def _read(self):
        for line in self.proc.stdout:
            f = [x.strip() for x in line.split(",")]
            if len(f) == 6:
                self.rows.append(f)

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if self.th is not None:
            self.th.join(timeout=5)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[2 + k] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(self.rows)}


def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_sample(graph, og, beam, max_active, n_utts, frames, seed_base=100):
    """Time the oracle C port (the reference algorithm) on host threads."""
    from oracle import oracle as O
    from paper_1804_03243_b200 import synthetic
    threads = cpu_threads()
    mats = [synthetic.hclg_matrix(seed_base + i, num_frames=frames) for i in range(n_utts)]
    t0 = time.perf_counter()
    tc, st, cnt = O.decode_batch_mt(graph, mats, beam, max_active=max_active, want_lattice=False,
                                    nthreads=threads, graph=og)
    dt = time.perf_counter() - t0
    return dt, n_utts * frames, int(cnt[:, 1].sum() + cnt[:, 4].sum()), threads, st


def run_reference(args, dist: Dist):
    """`--impl reference`: the reference decoder's algorithm on the host CPU."""
    if dist.rank != 0:
        dist.close()
        return
    from oracle import oracle as O
    from paper_1804_03243_b200 import synthetic
    graph = synthetic.hclg_graph(0, num_states=args.states)
    og = O.OracleGraph(graph)
    threads = cpu_threads()
    n = args.cpu_utts or threads
    for _ in range(args.warmup):
        cpu_sample(graph, og, 13.0, 7000, min(n, threads), 10)
    total_t, total_f, total_a = 0.0, 0, 0
    for k in range(args.steps):
        dt, fr, arcs, _, st = cpu_sample(graph, og, 13.0, 7000, n, args.cpu_frames, seed_base=100 + k * n)
        total_t += dt
        total_f += fr
        total_a += arcs
    v = total_f / total_t
    sample = f"{n} utterances x {args.cpu_frames} frames per step on {threads} threads (oracle C port)"
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": "frames/s", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total_t / args.steps,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic", "arcs_per_sec": total_a / total_t,
           "config": config_dict(args, note="CPU sample of the same workload"),
           "cpu_baseline": {"value": v, "unit": "frames/s", "cores": threads, "kind": "port",
                            "sample": sample},
           "e2e": {"value": v, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    dist.close()


def measure_configs(graph_c2, all_configs: bool) -> dict:
    """Frames/s of the other BASELINE.json configs through the public API
    (host numpy costs in, DecodeResult out; two warm-up calls, then the median of
    three timed calls, each a full decode_batch).
    C1: uniform 10k x 5 graph, 20 utterances x 300 frames, 1-best + lattice.
    C2: C2 HCLG, one utterance (one lane: the single-stream latency case).
    C3: C2 + exact lattice generation, pruning and finalisation.
    C5: the 50M-arc stress graph (only with --all-configs: it takes ~15 s to build)."""
    import paper_1804_03243_b200 as lb
    from paper_1804_03243_b200 import synthetic

    def run(name, graph, n_utts, want_lattice):
        d = synthetic.CONFIGS[name]["decode"]
        mats = [np.ascontiguousarray(synthetic.config_matrix(name, u).costs) for u in range(n_utts)]
        cfg = lb.DecodeConfig(beam=d["beam"], lattice_beam=d["lattice_beam"], max_active=d["max_active"],
                              max_lattice_arcs=50_000_000)
        for _ in range(2):   # workspace, pinned arena and host pages reach steady state
            lb.decode_batch(graph, mats, cfg, want_lattice=want_lattice)
        times = []
        for _ in range(3):
            t0 = time.perf_counter()
            res = lb.decode_batch(graph, mats, cfg, want_lattice=want_lattice)
            times.append(time.perf_counter() - t0)
        dt = float(np.median(times))
        frames = sum(m.shape[0] for m in mats)
        out = {"frames_per_s": frames / dt, "utterances": n_utts, "frames": frames, "seconds": dt,
               "seconds_all": times, "want_lattice": want_lattice}
        if want_lattice:
            out["lattice_arcs"] = int(sum(r.lattice.num_arcs for r in res))
        return out

    res = {"C1": run("C1", synthetic.config_graph("C1"), 20, True),
           "C2": run("C2", graph_c2, 1, False),
           "C3": run("C3", graph_c2, 1, True)}
    if all_configs:
        res["C5"] = run("C5", synthetic.config_graph("C5"), 1, False)
    res["note"] = "public API decode_batch, host costs, wall clock incl. H2D/D2H and host result assembly"
    return res


def config_dict(args, note=""):
    d = {"workload": "C4: sequence-parallel batch on the C2 HCLG graph (1-best, beam 13, max-active 7000)",
         "graph": f"hclg_graph(seed=0, states={args.states}), 3000 pdfs, acyclic epsilon depth<=4",
         "utts_per_step_per_gpu": args.utts, "frames_per_utt": args.frames, "beam": 13.0,
         "max_active": 7000, "lanes": args.lanes or "auto", "threads_per_cta": args.threads or 640,
         "ctas_per_lane": args.ctas or 2,
         "l2": "flushed between steps (256 MiB write); graph 0.36 GB > L2"}
    if note:
        d["note"] = note
    return d


def main(argv=None):
    args = parse_args(argv)
    dist = Dist(backend_gpu=args.impl == "ours")
    if args.impl == "reference":
        return run_reference(args, dist)

    import torch

    import paper_1804_03243_b200 as lb
    from paper_1804_03243_b200 import synthetic
    from paper_1804_03243_b200.resident import decode_batch_resident

    dev = dist.local
    torch.cuda.set_device(dev)
    graph = synthetic.hclg_graph(0, num_states=args.states)
    cfg = lb.DecodeConfig(beam=13.0, max_active=7000, lanes=args.lanes, threads_per_lane=args.threads,
                          ctas_per_lane=args.ctas, device=dev)
    lb.device_graph(graph, dev)
    U, T = args.utts, args.frames
    pool = 2 * U
    seeds = sorted({s for k in range(pool) for s in shard_seeds(dist.rank, k, U, pool)})
    host = {s: np.ascontiguousarray(synthetic.hclg_matrix(s, num_frames=T).costs) for s in seeds}
    resident = {s: torch.from_numpy(a).to(f"cuda:{dev}") for s, a in host.items()}
    # the other configs first, in a fresh process state (each has its own warm-up)
    configs = None
    if dist.rank == 0 and dist.world == 1 and not args.no_configs:
        configs = measure_configs(graph, args.all_configs)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{dev}")
    stream = torch.cuda.Stream(device=dev)     # the decode kernels and the timing events share it
    torch.cuda.set_stream(stream)

    def step_resident(k):
        outs, tm = decode_batch_resident(graph, [resident[s] for s in shard_seeds(dist.rank, k, U, pool)],
                                         cfg, stream=stream)
        bad = [o for o in outs if o["status"] != 0]
        if bad:
            raise RuntimeError(f"decode failed in bench step: {bad[0]}")
        return outs, tm

    for k in range(args.warmup):
        step_resident(k)
    torch.cuda.synchronize()
    clocks = ClockSampler(dev)
    clocks.start()
    dist.barrier()
    torch.cuda.synchronize()
    total_ms, kern_ms, launches, alg_bytes, arcs, host_ms = 0.0, 0.0, 0, 0, 0, 0.0
    for k in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        h0 = time.perf_counter()
        outs, tm = step_resident(args.warmup + k)
        host_ms += (time.perf_counter() - h0) * 1e3
        e1.record(stream)
        torch.cuda.synchronize()
        total_ms += e0.elapsed_time(e1)
        kern_ms += tm["decode_ms"]
        launches += tm["launches"]
        for o in outs:
            alg_bytes += bytes_of(o["counters"])
            arcs += int(o["counters"][1] + o["counters"][4])
    torch.cuda.synchronize()
    dist.barrier()
    ck = clocks.stop()
    t_max = dist.max(total_ms)
    frames_all = dist.sum(U * T * args.steps)
    arcs_all = dist.sum(arcs)
    value = frames_all / (t_max / 1e3)

    # ---- e2e through the public API (host matrices, H2D + D2H inside) ----
    e2e = None
    if not args.no_e2e:
        for k in range(1):
            lb.decode_batch(graph, [host[s] for s in shard_seeds(dist.rank, k, U, pool)], cfg,
                            want_lattice=False)
        torch.cuda.synchronize()
        dist.barrier()
        t_e2e = 0.0
        for k in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = lb.decode_batch(graph, [host[s] for s in shard_seeds(dist.rank, args.warmup + k, U, pool)],
                                  cfg, want_lattice=False)
            torch.cuda.synchronize()
            t_e2e += time.perf_counter() - t0
            assert all(r.total_cost == r.total_cost for r in res)
        t_e2e = dist.max(t_e2e)
        path_cap = 4 * T + 256
        e2e = {"value": frames_all / t_e2e, "unit": "frames/s",
               "h2d_bytes_per_step": U * T * 3000 * 8,
               "d2h_bytes_per_step": U * (8 * 4 + 4 * 8 + 8 * 8 + 4 * path_cap),
               "path": "paper_1804_03243_b200.decode_batch (host numpy f64 costs)"}

    # ---- roofline of the dominant kernel (decode_kernel) ----
    peaks = json.load(open(PEAKS)) if os.path.exists(PEAKS) else {}
    peak = peaks.get("hbm_gbs", 6650.0)
    achieved = alg_bytes / (kern_ms / 1e3) / 1e9
    traffic = None
    if os.path.exists(PROFILE_SUMMARY):
        traffic = json.load(open(PROFILE_SUMMARY)).get("dram_bytes_per_launch")
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic,
                "kernel": "decode_kernel", "alg_bytes_per_launch": alg_bytes / max(args.steps, 1),
                "kernel_ms_per_launch": kern_ms / max(args.steps, 1),
                "step_host_ms": host_ms / max(args.steps, 1),
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback"}

    cpu = None
    if dist.rank == 0 and dist.world == 1 and not args.no_cpu:
        from oracle import oracle as O
        og = O.OracleGraph(graph)
        n = args.cpu_utts or cpu_threads()
        dt, fr, _, threads, _ = cpu_sample(graph, og, 13.0, 7000, n, args.cpu_frames)
        cpu = {"value": fr / dt, "unit": "frames/s", "cores": threads, "kind": "port",
               "sample": f"{n} utterances x {args.cpu_frames} frames, oracle C port on {threads} threads"}

    if dist.rank == 0:
        out = {"metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": dist.world,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_max / args.steps,
               "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
               "data": "synthetic", "arcs_per_sec": arcs_all / (t_max / 1e3),
               "config": config_dict(args), "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
               "gpu_launches": launches, "clocks": ck, "configs_measured": configs}
        print(json.dumps(out), flush=True)
    dist.close()


if __name__ == "__main__":
    main()
