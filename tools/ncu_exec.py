"""Top SASS instructions by warp-level instructions executed (and shared
wavefronts) for one kernel of an ncu report.
Usage: python tools/ncu_exec.py rep.ncu-rep kernel_regex [N]"""
import csv
import io
import subprocess
import sys


def main(rep, kre, n=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kre,
                          "--print-source", "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "Address":
            if hdr:
                break
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    ex = "Instructions Executed"
    tot = sum(float(d[ex] or 0) for d in data) or 1
    print(f"{len(data)} SASS, {tot:.3e} warp instructions executed")
    for d in sorted(data, key=lambda d: -float(d[ex] or 0))[:n]:
        print(f"{100 * float(d[ex]) / tot:5.1f}%  {d['Address'][-5:]}  {d['Source'].strip()[:60]:60s} "
              f"thr/inst={float(d.get('Avg. Threads Executed') or 0):4.1f} smemwf={d.get('L1 Wavefronts Shared', '')}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 40)
