"""Summarise an ncu --set full report into profiles/ (JSON + text)."""
import csv
import io
import json
import subprocess
import sys

rep, out_json = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units, v = rows[0], rows[1], rows[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__cluster_dim_x",
        "smsp__thread_inst_executed_per_inst_executed.ratio",
        "lts__t_sectors_srcunit_tex_op_atom.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
        "lts__t_sectors_srcunit_tex_op_write.sum", "l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum",
        "l1tex__t_sectors_pipe_lsu_mem_local_op_st.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]
d = {}
for i, name in enumerate(h):
    if name in want:
        d[name] = {"value": v[i], "unit": units[i]}
def num(k):
    x = d[k]["value"].replace(",", "")
    u = d[k]["unit"]
    f = float(x)
    return f * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1.0}.get(u, 1)
summary = {"report": rep.split("/")[-1], "kernel": rows[2][h.index("Kernel Name")] if "Kernel Name" in h else None,
           "metrics": d,
           "dram_bytes_per_launch": num("dram__bytes_read.sum") + num("dram__bytes_write.sum"),
           "duration_s": num("gpu__time_duration.sum")}
json.dump(summary, open(out_json, "w"), indent=1)
print(json.dumps({k: summary[k] for k in ("dram_bytes_per_launch", "duration_s")}))
for k, x in d.items():
    print(f"{k:70s} {x['value']:>18s} {x['unit']}")
