"""Per-stage time and DRAM traffic of ONE product from an ncu launch list (gpu__time_duration.sum,
dram__bytes_read.sum, dram__bytes_write.sum; tools/one_product.py with reps products): launches are
assigned to bench.py's stages by kernel name and by their position relative to the product's tile
pass (conversion kernels before it are the forward conversion + encode, after it the decode + inverse
conversion).  The last product of the list is used.

usage: python tools/launch_stages.py LAUNCHES.csv BITS [--write profiles/traffic.json]
"""
import collections
import csv
import json
import sys

SCALE_T = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}
SCALE_B = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def launches(path):
    per = collections.OrderedDict()
    for r in csv.DictReader(l for l in open(path) if not l.startswith("==")):
        d = per.setdefault(r["ID"], {"name": r["Kernel Name"].split("(")[0]})
        v = float(r["Metric Value"].replace(",", ""))
        u = r["Metric Unit"]
        if r["Metric Name"] == "gpu__time_duration.sum":
            d["ms"] = v * SCALE_T.get(u, 1e-6)
        elif r["Metric Name"].startswith("dram__bytes_read"):
            d["rd"] = v * SCALE_B.get(u, 1)
        elif r["Metric Name"].startswith("dram__bytes_write"):
            d["wr"] = v * SCALE_B.get(u, 1)
    return [d for d in per.values() if "fpm::" in d["name"]]


def stages(ls):
    tiles = [k for k, d in enumerate(ls) if "fft_tile" in d["name"]]
    t = tiles[-1]  # the last product's tile pass
    lo = tiles[-2] + 1 if len(tiles) > 1 else 0
    # the last product starts after the previous product's last kernel (the one before this
    # product's first forward conversion kernel): walk back from the tile pass to the previous tile
    # pass, skipping the previous product's inverse part (everything up to its last conversion kernel
    # before a forward one is ambiguous, so count from the first kernel after the previous product's
    # final top_bit_fix / overflow-free tail: for one product per list lo = 0).
    out = collections.OrderedDict((k, {"ms": 0.0, "bytes": 0.0, "launches": 0}) for k in
                                  ("basiscvt+encode", "butterfly", "pointwise", "ibutterfly", "decode+ibasiscvt"))
    start = lo
    if len(tiles) > 1:  # skip the previous product's inverse tail: it ends with its top_bit_fix kernel
        for k in range(lo, t):
            if "top_bit_fix" in ls[k]["name"] or "store_product" in ls[k]["name"]:
                start = k + 1
    for k in range(start, len(ls)):
        d = ls[k]
        n = d["name"]
        if k == t or "fft_tile" in n:
            st = "pointwise"
        elif "fft_top" in n:
            st = "butterfly" if k < t else "ibutterfly"
        else:
            st = "basiscvt+encode" if k < t else "decode+ibasiscvt"
        o = out[st]
        o["ms"] += d.get("ms", 0.0)
        o["bytes"] += d.get("rd", 0.0) + d.get("wr", 0.0)
        o["launches"] += 1
    return out


def main():
    path, bits = sys.argv[1], int(sys.argv[2])
    out = stages(launches(path))
    print(f"{'stage':18s} {'launches':>8s} {'ms':>8s} {'GB':>8s} {'GB/s':>7s}")
    for k, o in out.items():
        print(f"{k:18s} {o['launches']:8d} {o['ms']:8.3f} {o['bytes'] / 1e9:8.3f} {o['bytes'] / (o['ms'] * 1e-3) / 1e9 if o['ms'] else 0:7.0f}")
    if "--write" in sys.argv:
        dst = sys.argv[sys.argv.index("--write") + 1]
        try:
            with open(dst) as f:
                t = json.load(f)
        except (OSError, ValueError):
            t = {}
        for k, o in out.items():
            t[f"{bits}:{k}"] = int(o["bytes"])
        with open(dst, "w") as f:
            json.dump(t, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
