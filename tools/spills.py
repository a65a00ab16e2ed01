"""Where does a kernel spill?  Local-memory SASS per source line (needs -lineinfo).
usage: python tools/spills.py <mangled-kernel-substring>"""
import re
import subprocess
import sys

pat = sys.argv[1] if len(sys.argv) > 1 else "decode_kernelILi768ELi2ELb0ELb0"
src = "paper_1804_03243_b200/csrc/latbeam_b200.cu"
subprocess.run(["nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-std=c++17",
                "-fmad=false", "-cubin", "-o", "/tmp/lb.cubin", src], check=True, capture_output=True)
dis = subprocess.run(["nvdisasm", "-g", "-c", "/tmp/lb.cubin"], capture_output=True, text=True).stdout
fn = cur = None
out = {}
for l in dis.split("\n"):
    m = re.match(r"\s*\.text\.(\S+):", l)
    if m:
        fn = m.group(1)
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
    if fn and pat in fn and re.search(r"\b(STL|LDL)", l):
        out.setdefault(cur, []).append(l.strip()[:50])
for k, v in sorted(out.items(), key=lambda x: str(x[0])):
    print(k, len(v), v[0])
