"""Opcode summary of the hot kernels' SASS (profiles/sass_r2.md): per kernel
instantiation of mpm_kernels.o, the counts of the memory / sync / fp64
opcodes and the TMA-class instructions verbatim.

    python tools/sass_summary.py [paper_2301_08343_b200/_lib/obj/mpm_kernels.o] > profiles/sass_r2.md
"""
import collections
import re
import subprocess
import sys

KEEP = re.compile(r"^(LDG|STG|LDS|STS|LDL|STL|RED|ATOM|BAR|SYNCS|UBLK|DADD|DFMA|DMUL|MUFU|CCTL|F2I|I2F|SHFL)")
TMA = re.compile(r"^(UBLK|SYNCS)")
KERNELS = ("k_g2p2g_gel", "k_grid_update_boxes", "k_ind_cols", "k_finalize", "k_p2g_gel_tile")


def main(obj):
    sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True,
                          check=True).stdout
    out = ["# SASS of the hot kernels (round 2, final kernels)", "",
           f"`cuobjdump -sass {obj}` (nvcc 12.9, `-gencode arch=compute_100a,code=sm_100a -O3`), "
           "per kernel instantiation: counts of the memory / sync / fp64 opcodes, then the "
           "TMA-class instructions verbatim (`python tools/sass_summary.py`).", "",
           "- `UBLKCP.S.G` = `cp.async.bulk` global->shared (the G2P velocity staging, one per "
           "z-row and array),",
           "- `UBLKRED.G.S.ADD.F64.RN` / `.ADD.U64` = `cp.reduce.async.bulk .add` shared->global "
           "(the P2G tile flush; U64 = fixed point in deterministic mode),",
           "- `SYNCS.*` = mbarrier init / arrive.expect_tx / try_wait (completion of the staging "
           "copies),",
           "- `REDG.E.ADD.F64.RN` / `REDG.E.ADD.64` = fire-and-forget global reductions "
           "(duplicate base cells, the indenter weight sums M_I; integer in deterministic mode).",
           ""]
    func = None
    counts = collections.OrderedDict()
    tma = {}
    for line in sass.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            func = m.group(1) if any(k in m.group(1) for k in KERNELS) else None
            if func:
                counts[func] = collections.Counter()
                tma[func] = []
            continue
        if not func:
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)([^;]*);", line)
        if not m:
            continue
        op = m.group(1)
        if KEEP.match(op):
            counts[func][op] += 1
        if TMA.match(op) and len(tma[func]) < 12:
            tma[func].append((op + m.group(2)).strip())
    for f, c in counts.items():
        out += [f"## `{f}`", "", "| opcode | count |", "|---|---|"]
        out += [f"| `{op}` | {n} |" for op, n in sorted(c.items())]
        if tma[f]:
            out += ["", "TMA / mbarrier instructions (first 12):", "", "```"] + tma[f] + ["```"]
        out.append("")
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "paper_2301_08343_b200/_lib/obj/mpm_kernels.o")
