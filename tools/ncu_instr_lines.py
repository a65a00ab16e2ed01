"""Warp instructions executed and stall samples per source line of an ncu report
(ncu --page source --print-source cuda,sass; needs -lineinfo).
usage: python tools/ncu_instr_lines.py report.ncu-rep [lane_frames] [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
lf = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
N = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, hdr, cur, src = None, None, None, {}
acc = {}
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] in ("File Name", "File Path"):
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None:
        continue
    if r[0]:
        cur = (fname, int(r[0]) if r[0].isdigit() else 0)
        src[cur] = r[1]
    if len(r) < 8 or not r[2]:
        continue
    d = dict(zip(hdr[4:], r[4:]))

    def f(k):
        try:
            return float(d.get(k, "0") or 0)
        except ValueError:
            return 0.0
    a = acc.setdefault(cur, [0.0, 0.0])
    a[0] += f("Instructions Executed")
    a[1] += f("Warp Stall Sampling (All Samples)")
tot_i = sum(v[0] for v in acc.values()) or 1
tot_s = sum(v[1] for v in acc.values()) or 1
print(f"warp instructions {tot_i:.4g} ({tot_i / lf:.0f} per lane-frame); stall samples {tot_s:.0f}")
for k, (i, s) in sorted(acc.items(), key=lambda x: -x[1][0])[:N]:
    print(f"{k[0]:>16}:{k[1]:<5} instr/lf={i / lf:8.0f} ({100 * i / tot_i:4.1f}%) samples={100 * s / tot_s:4.1f}%  "
          f"{src.get(k, '').strip()[:80]}")
