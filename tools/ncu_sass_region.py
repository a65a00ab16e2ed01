"""Stall samples of the SASS that belongs to a range of lb_kernels.cuh lines.
usage: python tools/ncu_sass_region.py report.ncu-rep first_line last_line [N]"""
import csv
import io
import subprocess
import sys

rep, lo, hi = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
N = int(sys.argv[4]) if len(sys.argv) > 4 else 40
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
    if a not in rows or (cur[0] == "lb_kernels.cuh"):
        rows[a] = (cur, r[3].strip(), d)
S = "Warp Stall Sampling (All Samples)"
tot = sum(float(d.get(S, 0) or 0) for _, _, d in rows.values())
sel = [(a, c, s, d) for a, (c, s, d) in sorted(rows.items()) if c[0] == "lb_kernels.cuh" and lo <= c[1] <= hi]
if sel:
    a0, a1 = sel[0][0], sel[-1][0]
    region = [(a, c, s, d) for a, (c, s, d) in sorted(rows.items()) if a0 <= a <= a1]
else:
    region = []
rs = sum(float(d.get(S, 0) or 0) for *_, d in region)
print(f"region {lo}-{hi}: {len(region)} instrs, {rs / tot * 100:.1f}% of samples")
stall = [k for k in (hdr or []) if k.startswith("stall_") and "Not Issued" not in k]
for a, c, s, d in sorted(region, key=lambda x: -float(x[3].get(S, 0) or 0))[:N]:
    v = float(d.get(S, 0) or 0)
    top = sorted(((float(d.get(k, 0) or 0), k[6:]) for k in stall), reverse=True)[:2]
    print(f"{v / tot * 100:5.2f}% {a & 0xfffff:05x} L{c[1]:<4d} exec={d.get('Instructions Executed'):>8s} {s[:52]:52s} "
          + " ".join(f"{k}:{x / max(v, 1) * 100:.0f}%" for x, k in top if x))
