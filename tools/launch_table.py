"""Summarise an ncu launch list (tools/gpu/launches.sh): per launch, or aggregated per kernel."""
import collections
import csv
import re
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, L = None, {}
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            e = L.setdefault(int(d["ID"]), {"name": d["Kernel Name"], "grid": d["Grid Size"]})
            e[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    return L


def short(n):
    m = re.search(r"igemm_kernel<__nv_bfloat16, (\d), (\d+), (\d), (\d)>", n)
    if m:
        return f"igemm {'FPROP DGRAD WGRAD'.split()[int(m.group(1))]} bn{m.group(2)} npw{m.group(3)} i2c{m.group(4)}"
    return re.sub(r"\(.*", "", n).replace("dsp::", "").replace("<unnamed>::", "")[-60:]


def main():
    L = load(sys.argv[1])
    mode = sys.argv[2] if len(sys.argv) > 2 else "launches"
    tot = sum(e.get("gpu__time_duration.sum", 0) for e in L.values()) / 1e3
    if mode == "launches":
        for k in sorted(L):
            e = L[k]
            t = e.get("gpu__time_duration.sum", 0) / 1e3
            b = (e.get("dram__bytes_read.sum", 0) + e.get("dram__bytes_write.sum", 0)) / 1e6
            print(f"{k:4d} {t:8.1f}us {b:8.1f}MB {b / t if t else 0:5.2f}TB/s {e['grid']:>14} {short(e['name'])}")
    else:
        agg = collections.defaultdict(lambda: [0.0, 0, 0.0])
        for e in L.values():
            a = agg[short(e["name"])]
            a[0] += e.get("gpu__time_duration.sum", 0) / 1e3
            a[1] += 1
            a[2] += (e.get("dram__bytes_read.sum", 0) + e.get("dram__bytes_write.sum", 0)) / 1e6
        for n, (t, c, b) in sorted(agg.items(), key=lambda x: -x[1][0]):
            print(f"{100 * t / tot:5.1f}% {t:9.1f}us n={c:4d} avg={t / c:8.1f}us {b / t if t else 0:5.2f}TB/s {n}")
    print(f"total {tot:.1f} us")


if __name__ == "__main__":
    main()
