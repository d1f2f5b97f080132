"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv).
Usage: python tools/launches.py gpurun_out/x_launches.csv [steps]"""
import collections
import csv
import sys


def main(path, steps=1):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for d in data:
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        k = d["Kernel Name"].split("(")[0][:70]
        tot[k] += float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1.0)
        cnt[k] += 1
    T = sum(tot.values())
    print(f"{'ms':>10} {'launches':>8} {'share':>6}  kernel   (all launches in the list; {T:.2f} ms total)")
    for k, v in sorted(tot.items(), key=lambda x: -x[1])[:30]:
        print(f"{v:10.3f} {cnt[k]:8d} {100 * v / T:5.1f}%  {k}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 1)
