"""Per-stage DRAM traffic (bytes read + written) of one product from an ncu report, for bench.py's
roofline "traffic" field: writes/updates profiles/traffic.json {"<bits>:<stage>": bytes}; with a
--set full report also the stage's pipe utilisation (duration-weighted over its launches) for the
roofline "ncu_pipes" field: profiles/pipes.json {"<bits>:<stage>": {metric: percent}}.

usage: python tools/ncu_traffic.py REPORT.ncu-rep BITS
The report must cover every launch of the stage (e.g. ncu --set full -k regex:fft_ -c N over
tools/one_product.py <lg> 1, after its warm-up product is skipped with --launch-skip)."""
import csv
import io
import json
import os
import subprocess
import sys

STAGE_OF = [("fft_top8_kernel<1", "ibutterfly"), ("fft_top8_kernel<0", "butterfly"), ("fft_tile_fused_kernel", "pointwise"), ("fft_tile_fused2_kernel", "pointwise"),
            ("fft_tile_tower_kernel", "pointwise"), ("fft_top4_kernel<1", "ibutterfly"),
            ("fft_top_kernel<1", "ibutterfly"), ("fft_top4_kernel<0", "butterfly"),
            ("fft_top_kernel<0", "butterfly"), ("fft_tile_kernel<0>", "butterfly"),
            ("encode_kernel", "encode"), ("decode_kernel", "decode")]


PIPES = {"issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
         "alu_pipe_pct": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
         "fma_pipe_pct": "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
         "lsu_pipe_pct": "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
         "shared_wavefronts_pct": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"}


def main(rep, bits):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          ",".join(["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"]
                                   + list(PIPES.values()))],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    units = rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    tot = {}
    pipes = {}  # stage -> (sum of duration, {key: sum of duration * pct})
    for r in rows[2:]:
        name = r[h.index("Kernel Name")]
        stage = next((st for key, st in STAGE_OF if key in name), None)
        if stage is None:
            continue
        b = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = h.index(m)
            b += float(r[i].replace(",", "")) * scale.get(units[i], 1)
        tot[stage] = tot.get(stage, 0.0) + b
        try:
            dur = float(r[h.index("gpu__time_duration.sum")].replace(",", ""))
            vals = {k: float(r[h.index(m)].replace(",", "")) for k, m in PIPES.items()}
        except (ValueError, IndexError):
            continue  # not a --set full capture
        d, acc = pipes.setdefault(stage, (0.0, {}))
        for k, v in vals.items():
            acc[k] = acc.get(k, 0.0) + dur * v
        pipes[stage] = (d + dur, acc)
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
    cur = {}
    if os.path.exists(path):
        with open(path) as f:
            cur = json.load(f)
    for st, b in tot.items():
        cur[f"{bits}:{st}"] = int(b)
    with open(path, "w") as f:
        json.dump(cur, f, indent=1, sort_keys=True)
    print(json.dumps({k: v for k, v in cur.items() if k.startswith(f"{bits}:")}))
    if pipes:
        ppath = os.path.join(os.path.dirname(path), "pipes.json")
        pc = {}
        if os.path.exists(ppath):
            with open(ppath) as f:
                pc = json.load(f)
        for st, (d, acc) in pipes.items():
            pc[f"{bits}:{st}"] = {k: round(v / d, 1) for k, v in acc.items()}
        with open(ppath, "w") as f:
            json.dump(pc, f, indent=1, sort_keys=True)
        print(json.dumps({k: v for k, v in pc.items() if k.startswith(f"{bits}:")}))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]))
