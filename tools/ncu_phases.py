"""Attribute ncu stall samples of decode_kernel to decode phases by SASS address:
each instruction inherits the phase of the nearest preceding lb_kernels.cuh line.
usage: python tools/ncu_phases.py report.ncu-rep"""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
src = open("paper_1804_03243_b200/csrc/lb_kernels.cuh").read().split("\n")
# phase ranges from function headers in lb_kernels.cuh
marks = []
for i, l in enumerate(src, 1):
    m = re.search(r"__device__ (?:double|void|bool|int) (emit|winners|max_active_cutoff|epsilon|aggregate|lattice|reset_touched)\(", l)
    if m:
        marks.append((i, m.group(1)))
    if "for_each_token_arc_batched(const" in l:
        marks.append((i, "tokarc_walk"))
    if l.startswith("decode_kernel(") or l.startswith("__global__"):
        marks.append((i, "kernel_body"))
marks.sort()


def phase_of(line):
    p = "other"
    for i, n in marks:
        if line >= i:
            p = n
    return p


out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, hdr = None, None
rows = []
cur_line = None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if r[0] == "Function Name":
        continue
    if r[0] != "":
        cur_line = (fname, int(r[0]))
        continue
    d = dict(zip(hdr[2:], r[2:]))
    try:
        rows.append((int(r[2], 16), cur_line, r[3], d))
    except ValueError:
        continue
rows.sort()
S = "Warp Stall Sampling (All Samples)"
tot = {}
last = "other"
allv = 0
for addr, (fn, ln), sass, d in rows:
    if fn == "lb_kernels.cuh":
        last = phase_of(ln)
    v = float(d.get(S, 0) or 0)
    allv += v
    key = last
    if "barrier" in sass.lower() or "BAR" in sass.split()[0:2].__str__() or "UCGABAR" in sass:
        key = last + "/barrier"
    tot[key] = tot.get(key, 0) + v
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{v / allv * 100:6.1f}%  {k}")
