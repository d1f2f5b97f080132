"""Per CUDA source line: warp instructions executed and stall samples for one
kernel of an ncu report (needs -lineinfo and --import-source on).
Usage: python tools/ncu_lines.py rep.ncu-rep kernel_regex [N]"""
import csv
import io
import subprocess
import sys


def main(rep, kre, n=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kre,
                          "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
    fname, hdr, data = "", None, []
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr and r[0] and len(r) >= 8:
            try:
                data.append((fname, int(r[0]), r[1], float(r[7] or 0), float(r[4] or 0)))
            except ValueError:
                pass
    ti = sum(d[3] for d in data) or 1
    ts = sum(d[4] for d in data) or 1
    print(f"warp insts {ti:.3e}, stall samples {ts:.0f}")
    for f, ln, src, ex, st in sorted(data, key=lambda d: -(d[3] / ti + d[4] / ts))[:n]:
        print(f"inst {100 * ex / ti:5.1f}%  stall {100 * st / ts:5.1f}%  {f}:{ln:<5d} {src.strip()[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 40)
