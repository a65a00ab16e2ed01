"""Benchmark: decoded frames/s (and arcs/s) of the B200 decoder on config C4.

Workload (BASELINE.json configs[3], "sequence-parallel batch: 64 concurrent
decode lanes per GPU, 4096 utterances sharded over 1/2/4/8 B200"): the C2/C3
HCLG-shaped graph (5M states, ~14.7M arcs, 3000 pdfs, acyclic epsilons), beam
13, max-active 7000, 1-best, T=300-frame utterances of i.i.d. U(0,5) f64
acoustic costs.  One step = the WHOLE 4096-utterance job: each rank takes its
longest-first shard of the utterance list (the same LPT split the multi-device
decode_batch uses) and decodes it in ONE call on 64 refilling decode lanes.
Total work is fixed as N grows, so `scaling` is "strong".

  value  frames/s with the cost matrices already resident in HBM (C-ABI
         lb_decode_batch_device, CUDA events on the launching stream, L2
         flushed between steps), max over ranks, whole box.
  e2e    the same metric through the public API `decode_batch` on host numpy
         matrices: the streamed pinned staging of the costs (H2D) and the D2H of
         the results are inside the timed region.

The synthetic utterances cycle through a pool of distinct seeded matrices (one
decode per utterance, nothing is cached between decodes).  `--ragged` draws
T uniformly from [100, 500] instead of 300 (the refilling scheduler's case).

`--impl reference` times the reference algorithm's CPU path instead (the
oracle/ C port of latbeam's decoder with the max-active extension, all host
threads), on the first utterances of the same list (same graph, same 300-frame
utterances).

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
D_PDFS = 3000


def bytes_of(c):
    """Algorithmic bytes of a decode, from the device counters
    [tokens, arcs scanned, candidates, eps frontier, eps arcs, eps candidates,
    tokens kept, lattice arcs]."""
    return (28 * c[0] + 16 * c[1] + 8 * c[2] + 28 * c[3] + 16 * c[4] + 8 * c[5] + 24 * c[6]
            + 16 * c[7])


def exp_bytes_of(c):
    """Arc-expansion bytes only (SURVEY.md §8(d) B_exp = 28 N + 16 N_scan + 8 N_cand)."""
    return 28 * c[0] + 16 * c[1] + 8 * c[2]


def _jsonable(o):
    if isinstance(o, np.generic):
        return o.item()
    raise TypeError(f"not JSON serialisable: {type(o).__name__}")


def parse_args(argv=None):
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--utts", type=int, default=int(os.environ.get("LB_BENCH_UTTS", 4096)),
                   help="utterances of the whole job (all ranks)")
    p.add_argument("--pool", type=int, default=256, help="distinct utterance matrices the job cycles through")
    p.add_argument("--frames", type=int, default=300)
    p.add_argument("--ragged", action="store_true", help="T ~ U[100, 500] per utterance")
    p.add_argument("--lanes", type=int, default=64, help="concurrent decode lanes per GPU")
    p.add_argument("--threads", type=int, default=0, help="threads per CTA of a lane")
    p.add_argument("--ctas", type=int, default=0, help="CTAs (thread-block cluster size) per lane")
    p.add_argument("--states", type=int, default=5_000_000)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--cpu-utts", type=int, default=0)
    p.add_argument("--cpu-frames", type=int, default=0, help="frames per CPU utterance (0 = the job's)")
    p.add_argument("--no-configs", action="store_true", help="skip the C1/C2/C3/ragged side measurements")
    p.add_argument("--no-phases", action="store_true", help="skip the phase-split (arc-expansion) run")
    p.add_argument("--all-configs", action="store_true", help="(default) also measure C5 (builds the 50M-arc graph)")
    p.add_argument("--no-c5", action="store_true", help="skip the C5 side measurements (~15 s graph build)")
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
            # LB_BENCH_BACKEND=gloo: the timing reductions over gloo (e.g. two ranks
            # sharing one GPU to exercise the multi-rank path; NCCL refuses that)
            backend = os.environ.get("LB_BENCH_BACKEND") or ("nccl" if backend_gpu else "gloo")
            if backend == "nccl":
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


def utterance_lengths(n: int, frames: int, ragged: bool, seed: int = 11) -> np.ndarray:
    if not ragged:
        return np.full(n, frames, dtype=np.int32)
    return np.random.default_rng(seed).integers(100, 501, size=n).astype(np.int32)


def rank_utterances(rank: int, world: int, n: int, lengths=None) -> list:
    """Utterances of the job this rank decodes: its shard of the longest-first
    split (decoder.shard_lpt == the C-ABI lb_shard_lpt of lb_decode_batch_multi)."""
    from paper_1804_03243_b200.decoder import split_batch
    T = np.full(n, 300, dtype=np.int32) if lengths is None else np.asarray(lengths, dtype=np.int32)
    return split_batch(T, world)[rank]


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


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def host_pool(n_pool: int, max_frames: int):
    """Distinct seeded matrices (hclg_matrix(100 + i)); utterance u uses pool[u % n_pool][:T_u]."""
    from paper_1804_03243_b200 import synthetic
    return [np.ascontiguousarray(synthetic.hclg_matrix(100 + i, num_frames=max_frames, num_pdfs=D_PDFS).costs)
            for i in range(n_pool)]


def cpu_sample(graph, og, beam, max_active, mats, threads):
    """Time the oracle C port (the reference algorithm) on host threads."""
    from oracle import oracle as O
    t0 = time.perf_counter()
    tc, st, cnt = O.decode_batch_mt(graph, mats, beam, max_active=max_active, want_lattice=False,
                                    nthreads=threads, graph=og)
    dt = time.perf_counter() - t0
    return dt, int(sum(m.shape[0] for m in mats)), int(cnt[:, 1].sum() + cnt[:, 4].sum()), st


def run_reference(args, dist: Dist):
    """`--impl reference`: the reference decoder's algorithm on the host CPU,
    one utterance per host thread (the reference's decode_batch pool), each step
    the next `threads` utterances of the job's list at their full length."""
    if dist.rank != 0:
        dist.close()
        return
    from oracle import oracle as O
    from paper_1804_03243_b200 import synthetic
    graph = synthetic.hclg_graph(0, num_states=args.states)
    og = O.OracleGraph(graph)
    threads = cpu_threads()
    n = args.cpu_utts or threads
    lengths = utterance_lengths(args.utts, args.frames, args.ragged)
    frames = args.cpu_frames or None
    pool = host_pool(min(args.pool, n * (args.steps + 1)), int(lengths.max()))

    def mats_of(k):
        ids = [(k * n + i) % args.utts for i in range(n)]
        return [pool[u % len(pool)][:(frames or lengths[u])] for u in ids]

    cpu_sample(graph, og, 13.0, 7000, [m[:20] for m in mats_of(0)], threads)   # warm-up (page-in)
    total_t, total_f, total_a = 0.0, 0, 0
    for k in range(args.steps):
        dt, fr, arcs, st = cpu_sample(graph, og, 13.0, 7000, mats_of(k), threads)
        total_t += dt
        total_f += fr
        total_a += arcs
    v = total_f / total_t
    sample = (f"{n} utterances x {frames or 'full-length'} frames of the job's list per step, one per host thread "
              f"({threads} threads, {cpu_model()}), oracle C port of the reference decoder")
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": "frames/s", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total_t / args.steps,
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic", "arcs_per_sec": total_a / total_t,
           "config": config_dict(args),
           "note": "CPU sample of the same workload (same graph, same 300-frame utterances of the job's list)",
           "cpu_baseline": {"value": v, "unit": "frames/s", "cores": threads, "kind": "port",
                            "sample": sample},
           "e2e": {"value": v, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out, default=_jsonable), flush=True)
    dist.close()


def measure_configs(graph_c2, all_configs: bool) -> dict:
    """Frames/s of the other BASELINE.json configs through the public API
    (host numpy costs in, DecodeResult out; two warm-up calls, then the median of
    three timed calls, each a full decode_batch).
    C1: uniform 10k x 5 graph, 20 utterances x 300 frames, 1-best + lattice.
    C2: C2 HCLG, one utterance (one lane: the single-stream latency case).
    C3: C2 + exact lattice generation, pruning and finalisation.
    C5: the 50M-arc stress graph (skipped with --no-c5: it takes ~15 s to build)."""
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
        g5 = synthetic.config_graph("C5")
        res["C5"] = run("C5", g5, 1, False)
        res["C5_batch"] = c5_batch_roofline(g5)
    res["note"] = "public API decode_batch, host costs, wall clock incl. H2D/D2H and host result assembly"
    return res


def c5_batch_roofline(g5, n_utts: int = 512, lanes: int = 64) -> dict:
    """C5 (50M arcs, ~1000 epsilon hubs of in-degree ~8.5k, beam 16, max-active
    20k) as a multi-utterance job (512 utterances cycling through 16 distinct
    matrices): HBM-resident costs, 64 refilling lanes; the decode kernel's
    algorithmic bytes over its event time."""
    import torch

    import paper_1804_03243_b200 as lb
    from paper_1804_03243_b200 import synthetic
    from paper_1804_03243_b200.resident import decode_batch_resident
    d = synthetic.CONFIGS["C5"]["decode"]
    pool = [torch.from_numpy(np.ascontiguousarray(synthetic.config_matrix("C5", u).costs)).cuda()
            for u in range(16)]
    tens = [pool[u % len(pool)] for u in range(n_utts)]
    cfg = lb.DecodeConfig(beam=d["beam"], max_active=d["max_active"], lanes=lanes)
    decode_batch_resident(g5, tens, cfg)
    torch.cuda.synchronize()
    outs, tm = decode_batch_resident(g5, tens, cfg)
    alg = sum(bytes_of(o["counters"]) for o in outs)
    peak = json.load(open(PEAKS)).get("hbm_gbs", 6650.0) if os.path.exists(PEAKS) else 6650.0
    frames = sum(int(t.shape[0]) for t in tens)
    ach = alg / (tm["decode_ms"] / 1e3) / 1e9
    return {"utterances": n_utts, "lanes": lanes, "frames": frames, "frames_per_s": frames / (tm["decode_ms"] / 1e3),
            "kernel_ms": tm["decode_ms"], "alg_bytes": alg, "achieved_gbs": ach, "frac": ach / peak,
            "status_ok": all(o["status"] == 0 for o in outs)}


def config_dict(args, note=""):
    d = {"workload": f"C4: one {args.utts}-utterance job on the C2 HCLG graph (1-best, beam 13, max-active 7000), "
                     f"{args.lanes} refilling decode lanes per GPU, utterances sharded longest-first over ranks",
         "graph": f"hclg_graph(seed=0, states={args.states}), 3000 pdfs, acyclic epsilon depth<=4",
         "utterances": args.utts,
         "frames_per_utt": "U[100,500]" if args.ragged else args.frames,
         "distinct_matrices": args.pool, "beam": 13.0, "max_active": 7000, "lanes_per_gpu": args.lanes,
         "threads_per_cta": args.threads or 640, "ctas_per_lane": args.ctas or 2,
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

    dev = dist.local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(dev)
    graph = synthetic.hclg_graph(0, num_states=args.states)
    cfg = lb.DecodeConfig(beam=13.0, max_active=7000, lanes=args.lanes, threads_per_lane=args.threads,
                          ctas_per_lane=args.ctas, device=dev)
    lb.device_graph(graph, dev)
    lengths = utterance_lengths(args.utts, args.frames, args.ragged)
    mine = rank_utterances(dist.rank, dist.world, args.utts, lengths)
    pool = host_pool(min(args.pool, args.utts), int(lengths.max()))
    host = [pool[u % len(pool)][:lengths[u]] for u in mine]
    dpool = [torch.from_numpy(m).to(f"cuda:{dev}") for m in pool]
    resident = [dpool[u % len(pool)][:lengths[u]] for u in mine]
    frames_mine = int(sum(int(lengths[u]) for u in mine))
    # the other configs first, in a fresh process state (each has its own warm-up)
    configs = None
    if dist.rank == 0 and dist.world == 1 and not args.no_configs:
        configs = measure_configs(graph, not args.no_c5)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{dev}")
    stream = torch.cuda.Stream(device=dev)     # the decode kernels and the timing events share it
    torch.cuda.set_stream(stream)

    def step_resident(tens, c=cfg):
        outs, tm = decode_batch_resident(graph, tens, c, stream=stream)
        bad = [o for o in outs if o["status"] != 0]
        if bad:
            raise RuntimeError(f"decode failed in bench step: {bad[0]}")
        return outs, tm

    for k in range(args.warmup):
        step_resident(resident)
    torch.cuda.synchronize()
    clocks = ClockSampler(dev)
    clocks.start()
    dist.barrier()
    torch.cuda.synchronize()
    total_ms, kern_ms, launches, alg_bytes, exp_bytes, arcs, host_ms = 0.0, 0.0, 0, 0, 0, 0, 0.0
    for k in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        h0 = time.perf_counter()
        outs, tm = step_resident(resident)
        host_ms += (time.perf_counter() - h0) * 1e3
        e1.record(stream)
        torch.cuda.synchronize()
        total_ms += e0.elapsed_time(e1)
        kern_ms += tm["decode_ms"]
        launches += tm["launches"]
        for o in outs:
            alg_bytes += bytes_of(o["counters"])
            exp_bytes += exp_bytes_of(o["counters"])
            arcs += int(o["counters"][1] + o["counters"][4])
    torch.cuda.synchronize()
    dist.barrier()
    ck = clocks.stop()
    t_max = dist.max(total_ms)
    frames_all = dist.sum(frames_mine * args.steps)
    arcs_all = dist.sum(arcs)
    value = frames_all / (t_max / 1e3)

    # ---- e2e through the public API (host matrices, streamed H2D + D2H inside) ----
    e2e = None
    if not args.no_e2e:
        lb.decode_batch(graph, host, cfg, want_lattice=False)
        torch.cuda.synchronize()
        dist.barrier()
        t_e2e = 0.0
        for k in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = lb.decode_batch(graph, host, cfg, want_lattice=False)
            torch.cuda.synchronize()
            t_e2e += time.perf_counter() - t0
            assert all(r.total_cost == r.total_cost for r in res)
        t_e2e = dist.max(t_e2e)
        path_cap = 4 * int(lengths.max()) + 256
        e2e = {"value": frames_all / t_e2e, "unit": "frames/s",
               "h2d_bytes_per_step": int(dist.sum(frames_mine * D_PDFS * 8)),
               "d2h_bytes_per_step": int(dist.sum(len(mine) * (8 * 4 + 4 * 8 + 8 * 8 + 4 * path_cap))),
               "path": "paper_1804_03243_b200.decode_batch (host numpy f64 costs, streamed pinned ring)"}

    # ---- roofline of the dominant kernel (decode_kernel) ----
    peaks = json.load(open(PEAKS)) if os.path.exists(PEAKS) else {}
    peak = peaks.get("hbm_gbs", 6650.0)
    achieved = alg_bytes / (kern_ms / 1e3) / 1e9
    traffic = None
    if os.path.exists(PROFILE_SUMMARY):   # ncu --set full capture of the same kernel, per utterance-frame
        prof = json.load(open(PROFILE_SUMMARY))
        traffic = prof.get("dram_bytes_per_frame", 0) * frames_mine or prof.get("dram_bytes_per_launch")
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic,
                "kernel": "decode_kernel", "alg_bytes_per_launch": alg_bytes / max(args.steps, 1),
                "kernel_ms_per_launch": kern_ms / max(args.steps, 1),
                "step_host_ms": host_ms / max(args.steps, 1),
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured)" if "hbm_gbs" in peaks else "fallback"}

    # ---- arc-expansion roofline: B_exp over the emit phase's share of the lanes' time ----
    if dist.rank == 0 and not args.no_phases:
        roofline["arc_expansion"] = phase_split(graph, resident, cfg, peak, step_resident)

    cpu = None
    if dist.rank == 0 and dist.world == 1 and not args.no_cpu:
        from oracle import oracle as O
        og = O.OracleGraph(graph)
        threads = cpu_threads()
        n = args.cpu_utts or threads
        frames = args.cpu_frames or None
        mats = [pool[u % len(pool)][:(frames or lengths[u])] for u in range(n)]
        dt, fr, _, _ = cpu_sample(graph, og, 13.0, 7000, mats, threads)
        cpu = {"value": fr / dt, "unit": "frames/s", "cores": threads, "kind": "port",
               "sample": f"{n} utterances x {frames or 'full-length'} frames of the job's list, "
                         f"oracle C port on {threads} threads ({cpu_model()})"}

    ragged = auto_lanes = None
    if dist.rank == 0 and dist.world == 1 and not args.no_configs and not args.ragged:
        ragged = ragged_variant(args, dpool, step_resident, flush)
        auto_lanes = auto_lanes_variant(resident, frames_mine, cfg, step_resident, flush)

    if dist.rank == 0:
        out = {"metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": dist.world,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_max / args.steps,
               "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
               "data": f"synthetic: seeded U(0,5) f64 costs, {args.utts} utterances cycling through "
                       f"{min(args.pool, args.utts)} distinct matrices",
               "arcs_per_sec": arcs_all / (t_max / 1e3),
               "config": config_dict(args), "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
               "gpu_launches": launches, "clocks": ck, "ragged_variant": ragged,
               "auto_lanes_variant": auto_lanes, "configs_measured": configs}
        print(json.dumps(out, default=_jsonable), flush=True)
    dist.close()


def phase_split(graph, resident, cfg, peak, step_resident, n_sub: int = 512) -> dict:
    """One unprofiled-clock phase-split run (LB_PHASE_PROFILE=1: the lane leader
    reads %globaltimer at each phase boundary) on the first n_sub utterances:
    the emit phase's lane-time share, and B_exp over the emit time per lane
    (lanes run concurrently, so the aggregate expansion bandwidth is
    sum(B_exp) / (sum of lane emit time / lanes))."""
    os.environ["LB_PHASE_PROFILE"] = "1"
    try:
        outs, tm = step_resident(resident[:n_sub])
    finally:
        del os.environ["LB_PHASE_PROFILE"]
    ph = tm["phases_ms"]
    lanes = min(int(cfg.lanes or 64), len(outs))
    bexp = sum(exp_bytes_of(o["counters"]) for o in outs)
    lane_ms = sum(ph.values())
    emit_ms_per_lane = ph["emit"] / lanes
    ach = bexp / (emit_ms_per_lane / 1e3) / 1e9
    return {"achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak, "b_exp": bexp,
            "emit_ms_per_lane": emit_ms_per_lane, "utterances": len(outs), "lanes": lanes,
            "phase_share": {k: v / lane_ms for k, v in ph.items() if lane_ms > 0},
            "kernel_ms_profiled": tm["decode_ms"],
            "definition": "B_exp = 28 N + 16 N_scan + 8 N_cand summed over the utterances; emit time = "
                          "sum over lanes of their emit-phase time / lanes (LB_PHASE_PROFILE run)"}


def auto_lanes_variant(resident, frames, cfg, step_resident, flush, steps: int = 2) -> dict:
    """The same job with the library's default lane count (lanes=0: one 2-CTA lane
    per SM pair, 74 on a B200) instead of the config's 64 -- not the headline,
    which keeps BASELINE.json's 64 lanes."""
    import dataclasses

    import torch
    c = dataclasses.replace(cfg, lanes=0)
    step_resident(resident, c)
    ms = 0.0
    for _ in range(steps):
        flush.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        step_resident(resident, c)
        e1.record()
        torch.cuda.synchronize()
        ms += e0.elapsed_time(e1)
    return {"frames_per_s": frames * steps / (ms / 1e3), "lanes": "auto (one 2-CTA lane per SM pair)",
            "steps": steps}


def ragged_variant(args, dpool, step_resident, flush, steps: int = 2) -> dict:
    """The same job with T ~ U[100, 500] (the refilling scheduler's case): frames/s
    with HBM-resident costs, to compare with the equal-length value."""
    import torch
    lengths = utterance_lengths(args.utts, args.frames, True)
    if int(lengths.max()) > int(dpool[0].shape[0]):
        from paper_1804_03243_b200 import synthetic
        dpool = [torch.from_numpy(np.ascontiguousarray(
            synthetic.hclg_matrix(100 + i, num_frames=int(lengths.max()), num_pdfs=D_PDFS).costs)).cuda()
            for i in range(len(dpool))]
    tens = [dpool[u % len(dpool)][:lengths[u]] for u in range(args.utts)]
    step_resident(tens)
    ms = 0.0
    for _ in range(steps):
        flush.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        step_resident(tens)
        e1.record()
        torch.cuda.synchronize()
        ms += e0.elapsed_time(e1)
    frames = int(lengths.sum()) * steps
    return {"frames_per_s": frames / (ms / 1e3), "utterances": args.utts, "frames_per_step": int(lengths.sum()),
            "lengths": "U[100,500]", "steps": steps}


if __name__ == "__main__":
    main()
