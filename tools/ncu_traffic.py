"""Per-kernel DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum, per
launch, averaged over the captured launches) and shared-memory wavefronts
(l1tex__data_pipe_lsu_wavefronts_mem_shared) from an ncu --set full report,
written as JSON for bench.py's roofline "traffic" / "shared_memory" fields.

    python tools/ncu_traffic.py gpurun_out/prof.ncu-rep > profiles/traffic.json
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, data = rows[0], rows[2:]
    name_i = hdr.index("Kernel Name")
    ri, wi = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
    ti = hdr.index("gpu__time_duration.sum")
    # units can differ per row in ncu's CSV; re-query with explicit base units
    raw2 = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--print-units", "base"],
                          capture_output=True, text=True, check=True).stdout
    rows2 = list(csv.reader(io.StringIO(raw2)))[2:]
    si = hdr.index("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum")
    sp = hdr.index("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed")
    acc = defaultdict(lambda: [0.0, 0.0, 0, 0.0, 0.0])
    for r in rows2:
        name = r[name_i].split("(")[0].replace("void ", "").split("<")[0].strip()
        acc[name][0] += float(r[ri]) + float(r[wi])
        acc[name][1] += float(r[ti])
        acc[name][2] += 1
        acc[name][3] += float(r[si] or 0)
        acc[name][4] += float(r[sp] or 0)
    out = {k: {"dram_bytes_per_launch": v[0] / v[2], "ncu_time_ns": v[1] / v[2], "launches": v[2],
               "shared_wavefronts_per_launch": v[3] / v[2],
               "shared_wavefronts_pct_of_peak": v[4] / v[2], "report": path}
           for k, v in acc.items()}
    json.dump(out, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main(sys.argv[1])
