"""Summarise ncu captures of the secondary paths (exact SIMT kernel, large-k
kernels) into one markdown table (run here, no GPU needed).

    python tools/summarize_secondary.py <out.md> <label>=<rep.ncu-rep> ...
"""
import sys

from summarize_ncu import METRICS, raw

EXTRA = {
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "FMA pipe active %",
    "smsp__inst_executed.sum": "warp instructions",
}


def main():
    out = sys.argv[1]
    cols = dict(METRICS)
    cols.update(EXTRA)
    lines = ["| capture | kernel | " + " | ".join(cols.values()) + " |",
             "|---|---|" + "---|" * len(cols)]
    for arg in sys.argv[2:]:
        label, rep = arg.split("=", 1)
        data, units = raw(rep)
        for d in data:
            name = d.get("Kernel Name", "?").split("(")[0].replace("(anonymous namespace)::", "")
            vals = [f"{d.get(m, '')} {units.get(m, '')}".strip() for m in cols]
            lines.append(f"| {label} | {name} | " + " | ".join(vals) + " |")
    with open(out, "w") as f:
        f.write("# ncu --set full, secondary paths (one launch each)\n\n" + "\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
