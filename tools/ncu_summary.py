"""Summarise an ncu report (per-kernel key metrics) as markdown.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep > profiles/<name>.md
"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "DRAM rd"),
    ("dram__bytes_write.sum", "DRAM wr"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
    ("launch__registers_per_thread", "regs"),
    ("smsp__sass_inst_executed_op_global_red.sum", "RED instr"),
]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    cols = [(hdr.index(m), label, units[hdr.index(m)]) for m, label in METRICS if m in hdr]
    name_i = hdr.index("Kernel Name")
    print(f"ncu --set full summary of `{path}`\n")
    print("| kernel | " + " | ".join(f"{l} ({u})" if u else l for _, l, u in cols) + " |")
    print("|---|" + "---|" * len(cols))
    for r in data:
        name = r[name_i].split("(")[0].replace("void ", "")
        print(f"| {name} | " + " | ".join(r[i] for i, _, _ in cols) + " |")


if __name__ == "__main__":
    main(sys.argv[1])
