"""Top SASS instructions by warp-stall samples for one kernel of an ncu report
(needs -lineinfo builds and --import-source).  Usage:
python tools/ncu_hot.py rep.ncu-rep kernel_regex [N]"""
import csv
import io
import subprocess
import sys


def main(rep, kre, n=30):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kre,
                          "--print-source", "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = None
    data = []
    for r in rows:
        if r and r[0] == "Address":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            try:
                float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
            except ValueError:
                continue
            data.append(dict(zip(hdr, r)))
        if len(data) and r and r[0] == "Kernel Name":
            break
    key = "Warp Stall Sampling (All Samples)"
    tot = sum(float(d[key] or 0) for d in data) or 1
    print(f"{len(data)} SASS instructions, {tot:.0f} stall samples")
    for d in sorted(data, key=lambda d: -float(d[key] or 0))[:n]:
        print("%5.1f%%  %s  %-58s exec=%s" % (100 * float(d[key] or 0) / tot, d["Address"], d["Source"][:58],
                                             d.get("Instructions Executed", "")))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 30)
