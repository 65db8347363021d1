"""Summarise ncu captures into profiles/ (run here, no GPU needed).

    python tools/summarize_ncu.py <full.ncu-rep> <launches.csv> <out_prefix>

Writes <out_prefix>_kernels.md (key metrics per captured kernel, including the
per-launch DRAM traffic bench.py reports as roofline.traffic),
<out_prefix>_traffic.json and <out_prefix>_launches.md (share of step time
per kernel from the cold-cache launch list)."""
import csv
import io
import json
import subprocess
import sys
from collections import OrderedDict, defaultdict

METRICS = OrderedDict([
    ("gpu__time_duration.sum", "duration"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active %"),
    ("sm__inst_executed_pipe_tensor.avg.pct_of_peak_sustained_active", "tensor pipe inst %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum", "TMA load bytes"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
])


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [dict(zip(hdr, r)) for r in rows[2:]], dict(zip(hdr, units))


def main():
    rep, launches, prefix = sys.argv[1], sys.argv[2], sys.argv[3]
    data, units = raw(rep)
    lines = ["| kernel | " + " | ".join(METRICS.values()) + " |",
             "|---|" + "---|" * len(METRICS)]
    traffic = {}
    for d in data:
        name = d.get("Kernel Name", "?").split("(")[0].replace("(anonymous namespace)::", "")
        vals = []
        for m in METRICS:
            v = d.get(m, "")
            u = units.get(m, "")
            vals.append(f"{v} {u}".strip())
        lines.append(f"| {name} | " + " | ".join(vals) + " |")
        try:
            def tob(m):
                v = float(d[m].replace(",", ""))
                u = units.get(m, "byte")
                return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
            traffic.setdefault(name, []).append(tob("dram__bytes_read.sum") + tob("dram__bytes_write.sum"))
        except Exception:
            pass
    with open(prefix + "_kernels.md", "w") as f:
        f.write(f"# ncu --set full summary ({rep.split('/')[-1]})\n\n" + "\n".join(lines) + "\n")
    with open(prefix + "_traffic.json", "w") as f:
        json.dump({k: sum(v) / len(v) for k, v in traffic.items()}, f, indent=1)
    # launch list shares
    rows = list(csv.reader(open(launches)))
    hdr = None
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") != "gpu__time_duration.sum":
                continue
            name = d["Kernel Name"].split("(")[0].replace("(anonymous namespace)::", "")
            v = float(d["Metric Value"].replace(",", ""))
            scale = {"ns": 1e-3, "us": 1, "usecond": 1, "msecond": 1e3, "ms": 1e3}.get(d["Metric Unit"], 1e-3)
            tot[name] += v * scale
            cnt[name] += 1
    total = sum(tot.values())
    out = ["# launch list (ncu --metrics gpu__time_duration.sum --clock-control none)", "",
           "Cold-cache, serialised per-launch times: compare shares, not absolutes.", "",
           "| kernel | launches | total us | mean us | share |", "|---|---|---|---|---|"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        out.append(f"| {k} | {cnt[k]} | {v:.1f} | {v / cnt[k]:.1f} | {100 * v / total:.1f}% |")
    with open(prefix + "_launches.md", "w") as f:
        f.write("\n".join(out) + "\n")
    print(open(prefix + "_kernels.md").read())
    print("\n".join(out))


if __name__ == "__main__":
    main()
