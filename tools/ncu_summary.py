"""Condenses an ncu report into the summary committed under profiles/:
per kernel launch the duration, DRAM bytes (traffic), throughput fractions,
occupancy, L1/L2 hit rates, shared-atomic wavefronts and the top warp stall
reasons.  Usage: python tools/ncu_summary.py gpurun_out/x.ncu-rep > profiles/x.md"""
import csv
import io
import subprocess
import sys

RAW = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_%peak"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_%"),
    ("l1tex__t_sector_hit_rate.pct", "l1_hit_%"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex_%peak"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2_%peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_%"),
    ("smsp__inst_executed.sum", "warp_insts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum", "smem_atom_wavefronts"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    print(f"# ncu summary: `{path}`\n")
    for row in rows[2:]:
        name = row[hdr.index("Kernel Name")]
        print(f"## {name[:120]}\n")
        print("| metric | value | unit |\n|---|---|---|")
        for key, label in RAW:
            if key in hdr:
                i = hdr.index(key)
                print(f"| {label} (`{key}`) | {row[i]} | {units[i]} |")
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
                try:
                    stalls.append((float(row[i]), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(v for v, _ in stalls) or 1.0
        print("\ntop stall reasons (pc samples): " + ", ".join(
            f"{h} {100 * v / tot:.0f}%" for v, h in sorted(stalls, reverse=True)[:6]) + "\n")


if __name__ == "__main__":
    main(sys.argv[1])
