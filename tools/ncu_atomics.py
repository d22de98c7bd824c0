"""Per-kernel L2 reduction / atomic counters from an ncu report taken with
the metrics below (averaged per launch), as JSON (merged into
profiles/traffic.json by the caller) and as a markdown table.

    ncu --metrics <METRICS> --clock-control none -k regex:<kernels> -c N -o red \\
        python tools/profile_run.py config2a 2
    python tools/ncu_atomics.py gpurun_out/red.ncu-rep [profiles/atomics_r2.md]
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "lts__t_requests_op_red.sum", "lts__t_sectors_op_red.sum",
    "lts__t_requests_op_atom.sum", "lts__t_sectors_op_atom.sum",
    "lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sectors.sum",
    "sm__sass_inst_executed_op_tma_red.sum", "sm__sass_inst_executed_op_tma_ld.sum",
    "smsp__sass_inst_executed_op_global_red.sum",
    "l1tex__m_l1tex2xbar_write_bytes_mem_global_op_red.sum",
]


def main(path, md=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--print-units", "base"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, data = rows[0], rows[2:]
    name_i = hdr.index("Kernel Name")
    cols = [(m, hdr.index(m)) for m in METRICS if m in hdr]
    acc = defaultdict(lambda: defaultdict(float))
    cnt = defaultdict(int)
    for r in data:
        name = r[name_i].split("(")[0].replace("void ", "").split("<")[0].strip()
        cnt[name] += 1
        for m, i in cols:
            try:
                acc[name][m] += float(r[i].replace(",", ""))
            except ValueError:
                pass
    out = {k: {m: v / cnt[k] for m, v in d.items()} | {"launches": cnt[k], "report": path}
           for k, d in acc.items()}
    json.dump(out, sys.stdout, indent=1)
    print()
    if md:
        with open(md, "w") as f:
            f.write(f"# L2 reduction / atomic counters per launch (`{path}`)\n\n")
            f.write("| kernel | " + " | ".join(m for m, _ in cols) + " |\n")
            f.write("|---|" + "---|" * len(cols) + "\n")
            for k, d in out.items():
                f.write(f"| {k} | " + " | ".join(f"{d.get(m, 0):.4g}" for m, _ in cols) + " |\n")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
