"""Per-kernel table from an ncu --csv launch list with gpu__time_duration.sum and
dram__bytes_read.sum / dram__bytes_write.sum: launches, total ms, GB read/written, achieved GB/s.
usage: python tools/kernel_table.py LAUNCHES.csv [substring-filter]"""
import collections
import csv
import sys

SCALE_T = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}
SCALE_B = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def main(path, filt=""):
    rows = [r for r in csv.DictReader(l for l in open(path) if not l.startswith("=="))]
    per = collections.OrderedDict()
    for r in rows:
        key = (r["ID"], r["Kernel Name"].split("(")[0][:64])
        d = per.setdefault(key, {})
        v = float(r["Metric Value"].replace(",", ""))
        u = r["Metric Unit"]
        if r["Metric Name"] == "gpu__time_duration.sum":
            d["ms"] = v * SCALE_T.get(u, 1e-6)
        elif r["Metric Name"].startswith("dram__bytes_read"):
            d["rd"] = v * SCALE_B.get(u, 1)
        elif r["Metric Name"].startswith("dram__bytes_write"):
            d["wr"] = v * SCALE_B.get(u, 1)
    agg = collections.OrderedDict()
    for (_, name), d in per.items():
        if filt not in name:
            continue
        a = agg.setdefault(name, [0, 0.0, 0.0, 0.0])
        a[0] += 1
        a[1] += d.get("ms", 0)
        a[2] += d.get("rd", 0)
        a[3] += d.get("wr", 0)
    tot = [0, 0.0, 0.0, 0.0]
    print(f"{'launches':>8} {'ms':>9} {'GB rd':>8} {'GB wr':>8} {'GB/s':>8}  kernel")
    for name, (n, ms, rd, wr) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{n:8d} {ms:9.3f} {rd / 1e9:8.3f} {wr / 1e9:8.3f} {(rd + wr) / (ms * 1e-3) / 1e9 if ms else 0:8.0f}  {name}")
        tot = [tot[0] + n, tot[1] + ms, tot[2] + rd, tot[3] + wr]
    print(f"{tot[0]:8d} {tot[1]:9.3f} {tot[2] / 1e9:8.3f} {tot[3] / 1e9:8.3f} {(tot[2] + tot[3]) / (tot[1] * 1e-3) / 1e9 if tot[1] else 0:8.0f}  total")


if __name__ == "__main__":
    main(*sys.argv[1:])
