"""Per-kernel summary of an ncu --set full report (the profiles/*_ncu_full_summary.txt tables):
launches, ms, DRAM GB and GB/s, and duration-weighted issue / ALU / FMA / shared-wavefront / L1 /
occupancy percentages.  usage: python tools/ncu_summary.py REPORT.ncu-rep"""
import collections
import csv
import io
import subprocess
import sys

M = {"dur": "gpu__time_duration.sum", "rd": "dram__bytes_read.sum", "wr": "dram__bytes_write.sum",
     "issue": "smsp__issue_active.avg.pct_of_peak_sustained_active",
     "ALU": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
     "FMA": "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
     "smem": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
     "L1": "l1tex__throughput.avg.pct_of_peak_sustained_active",
     "occ": "sm__warps_active.avg.pct_of_peak_sustained_active"}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0,
         "ns": 1e-6, "us": 1e-3, "ms": 1.0, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv", "--metrics", ",".join(M.values())],
                     capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, units = rows[0], rows[1]
agg = collections.OrderedDict()
for r in rows[2:]:
    name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "").split("::")[-1]
    v = {}
    for k, m in M.items():
        i = h.index(m)
        v[k] = float(r[i].replace(",", "")) * SCALE.get(units[i], 1)
    a = agg.setdefault(name, collections.Counter())
    a["n"] += 1
    for k in ("dur", "rd", "wr"):
        a[k] += v[k]
    for k in ("issue", "ALU", "FMA", "smem", "L1", "occ"):
        a[k] += v[k] * v["dur"]
print(f"{'kernel':26s} {'n':>2s} {'ms':>8s} {'DRAM GB':>7s} {'GB/s':>6s}" +
      "".join(f" {k:>6s}" for k in ("issue", "ALU", "FMA", "smem", "L1", "occ")))
for name, a in sorted(agg.items(), key=lambda x: -x[1]["dur"]):
    gb = (a["rd"] + a["wr"]) / 1e9
    print(f"{name[:26]:26s} {a['n']:2d} {a['dur']:8.3f} {gb:7.2f} {gb / (a['dur'] / 1e3):6.0f}" +
          "".join(f" {a[k] / a['dur']:6.1f}" for k in ("issue", "ALU", "FMA", "smem", "L1", "occ")))
