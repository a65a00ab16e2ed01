"""Per-source-line hot spots of an ncu report (needs -lineinfo): stall samples,
local-memory (spill) sectors and global sectors, top N lines.
usage: python tools/ncu_lines.py report.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, hdr, lines = None, None, []
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "" or r[0] == "Function Name":
        continue
    d = dict(zip(hdr[2:], r[2:]))
    lines.append((fname, r[0], r[1], d))


def f(d, k):
    try:
        return float(d.get(k, "0") or 0)
    except ValueError:
        return 0.0


S = "Warp Stall Sampling (All Samples)"
tot = sum(f(d, S) for *_, d in lines) or 1
loc = sum(f(d, "L2 Theoretical Sectors Local") for *_, d in lines)
glb = sum(f(d, "L2 Theoretical Sectors Global") for *_, d in lines)
print(f"samples={tot:.0f}  local sectors={loc:.3g}  global sectors={glb:.3g}")
stall_cols = [k for k in (hdr or []) if k.startswith("stall_") and "Not Issued" not in k]
for fn, ln, src, d in sorted(lines, key=lambda x: -f(x[3], S))[:N]:
    top = sorted(((f(d, k), k[6:]) for k in stall_cols), reverse=True)[:2]
    ts = ",".join(f"{k}:{v / max(f(d, S), 1) * 100:.0f}%" for v, k in top if v)
    print(f"{f(d, S) / tot * 100:5.1f}% {fn}:{ln:>4s} loc={f(d, 'L2 Theoretical Sectors Local'):.2g} "
          f"glb={f(d, 'L2 Theoretical Sectors Global'):.2g} [{ts}] {src.strip()[:80]}")
