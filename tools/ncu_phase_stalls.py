"""Stall-reason breakdown per decode phase (SASS address attribution, see ncu_phases.py).
usage: python tools/ncu_phase_stalls.py report.ncu-rep"""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
src = open("paper_1804_03243_b200/csrc/lb_kernels.cuh").read().split("\n")
marks = []
for i, l in enumerate(src, 1):
    m = re.search(r"__device__ (?:__noinline__ )?(?:double|void|bool|int) (emit|winners|max_active_cutoff|epsilon|"
                  r"aggregate|flush_tokens|lattice|reset_touched|fix_preds)\(", l)
    if m:
        marks.append((i, m.group(1)))
    if "for_each_token_arc_batched(const" in l:
        marks.append((i, "walk"))
    if l.startswith("decode_kernel(") or l.startswith("prune_kernel(") or l.startswith("expand_kernel("):
        marks.append((i, "kernel"))
marks.sort()


def ph(line):
    p = "pre"
    for i, n in marks:
        if line >= i:
            p = n
    return p


out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
hdr = cur = None
rows = {}
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if r[0] == "Function Name":
        continue
    if r[0] != "":
        cur = (f, int(r[0]))
        continue
    d = dict(zip(hdr[2:], r[2:]))
    try:
        a = int(r[2], 16)
    except ValueError:
        continue
    if a not in rows or cur[0] == "lb_kernels.cuh":
        rows[a] = (cur, r[3].strip(), d)
stall = [k for k in hdr if k.startswith("stall_") and "Not Issued" not in k]
agg = {}
last = "pre"
tot = 0.0
for a, (c, s, d) in sorted(rows.items()):
    if c[0] == "lb_kernels.cuh":
        last = ph(c[1])
    x = agg.setdefault(last, {})
    for k in stall:
        v = float(d.get(k, 0) or 0)
        x[k[6:]] = x.get(k[6:], 0) + v
        tot += v
    x["_inst"] = x.get("_inst", 0) + float(d.get("Instructions Executed", 0) or 0)
for p, x in sorted(agg.items(), key=lambda kv: -sum(v for k, v in kv[1].items() if k != "_inst")):
    s = sum(v for k, v in x.items() if k != "_inst")
    if s / tot < 0.005:
        continue
    top = sorted(((v, k) for k, v in x.items() if k != "_inst"), reverse=True)[:6]
    print(f"{p:18s} {s / tot * 100:5.1f}% inst={x['_inst']:.3g}  " + " ".join(f"{k}:{v / s * 100:.0f}%" for v, k in top))
