"""Per CUDA source line: shared-memory wavefronts and executed instructions
for one kernel of an ncu report.  Usage: python tools/ncu_smem_lines.py rep kernel_regex [N]"""
import csv
import io
import subprocess
import sys


def main(rep, kre, n=20):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kre,
                          "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
    hdr, data, fname = None, [], ""
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
        elif r[0] == "Line No":
            hdr = r
        elif hdr and r[0] and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            d["file"] = fname
            data.append(d)
    k = "L1 Wavefronts Shared"
    tot = sum(float(d[k] or 0) for d in data) or 1
    print(f"shared wavefronts {tot:.3e}")
    for d in sorted(data, key=lambda d: -float(d[k] or 0))[:n]:
        print(f"{100 * float(d[k] or 0) / tot:5.1f}%  {d['file']}:{d['Line No']:<5} {d['Source'].strip()[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 20)
