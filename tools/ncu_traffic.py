"""Writes profiles/ncu_traffic.json from ncu --set full reports of the SAME
column batch's product kernels (bench.py reads it into roofline.traffic):
DRAM bytes read + written summed over the kernels captured in each report,
next to that batch's algorithmic bytes (roofline.alg_bytes_per_batch[batch]
of a bench line from the same build).

    python tools/ncu_traffic.py BENCH_LINE.json KEY=REPORT:BATCH[:BENCHKEY] ...
    (KEY e.g. or_and_u8; BENCHKEY = min_plus_i32 to read the sub-line)"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def kernels(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], dict(zip(rows[0], rows[1]))
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-6, "us": 1e-3, "usecond": 1e-3,
             "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6, "s": 1e3, "second": 1e3}
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        if not d.get("Kernel Name"):
            continue

        def f(k):
            v = d.get(k, "0").replace(",", "")
            try:
                return float(v) * scale.get(units.get(k, ""), 1.0)
            except ValueError:
                return 0.0
        res.append({"kernel": d["Kernel Name"].split("(")[0], "ms": f("gpu__time_duration.sum"),
                    "dram_bytes": f("dram__bytes_read.sum") + f("dram__bytes_write.sum")})
    return res


def main():
    line = json.loads([ln for ln in open(sys.argv[1]) if ln.startswith("{")][-1])
    out = {}
    for spec in sys.argv[2:]:
        key, rest = spec.split("=", 1)
        parts = rest.split(":")
        rep, batch = parts[0], int(parts[1])
        sub = line[parts[2]] if len(parts) > 2 else line
        ks = kernels(rep)
        alg = sub["roofline"]["alg_bytes_per_batch"][batch]
        tot = sum(k["dram_bytes"] for k in ks)
        out[key] = {"dram_bytes_per_launch": int(tot), "alg_bytes_same_batch": int(alg), "batch": batch,
                    "traffic_over_alg": round(tot / alg, 3) if alg else None,
                    "kernels": [{"kernel": k["kernel"], "ms": round(k["ms"], 3), "dram_bytes": int(k["dram_bytes"])}
                                for k in ks],
                    "source": f"ncu --set full of the product kernels of column batch {batch} ({os.path.basename(rep)})"}
    with open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
