"""Summarize ncu artifacts into profiles/: per-kernel table from a `--set full`
report and per-launch shares from a `gpu__time_duration` launch list.

    python profiles/summarize_ncu.py gpurun_out/step_r1.ncu-rep gpurun_out/launches_r1.csv > profiles/r1_summary.md
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "LSU ld sectors"),
    ("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "LSU ld requests"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
]


def traffic_json(path, out):
    """Per-kernel DRAM bytes per launch (read + write) from a --set full report."""
    import json
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    acc = defaultdict(list)
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")
        b = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = hdr.index(m)
            b += float(r[i].replace(",", "")) * scale[units[i]]
        acc[name].append(b)
    json.dump({"source": path, "metric": "dram__bytes_read.sum + dram__bytes_write.sum",
               "kernels": {k: {"dram_bytes_per_launch": sum(v) / len(v), "launches": len(v)}
                           for k, v in acc.items()}}, open(out, "w"), indent=1)


def full_report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    print(f"## ncu --set full: {path}\n")
    print("| kernel | " + " | ".join(n for _, n in METRICS) + " | LSU sectors/request | top stalls |")
    print("|---" * (len(METRICS) + 3) + "|")
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")
        cells = []
        for m, _ in METRICS:
            if m in hdr:
                i = hdr.index(m)
                cells.append(f"{r[i]} {units[i]}".strip())
            else:
                cells.append("-")
        st = [(h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""),
               float(r[i] or 0)) for i, h in enumerate(hdr)
              if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio")]
        st = ", ".join(f"{n} {v:.2f}" for n, v in sorted(st, key=lambda x: -x[1])[:3])
        spr = "-"
        try:
            sec = float(r[hdr.index("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum")].replace(",", ""))
            req = float(r[hdr.index("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum")].replace(",", ""))
            spr = f"{sec / req:.2f}" if req else "-"
        except (ValueError, IndexError):
            pass
        print(f"| {name} | " + " | ".join(cells) + f" | {spr} | {st} |")
    print()


STEP_KERNELS = ("k_prepare", "k_score", "k_select", "k_worklist", "k_attend", "k_merge_units", "k_append", "k_approx", "k_merge_chunks", "k_merge_runs")


def launch_list(path):
    lines = [ln for ln in open(path) if ln.startswith('"')]  # drop ncu's ==PROF== chatter
    rows = list(csv.DictReader(lines))
    t = defaultdict(list)
    by = defaultdict(dict)
    for r in rows:
        key = (r["ID"], r["Kernel Name"].split("(")[0].replace("void ", ""))
        by[key][r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    for (i, name), m in by.items():
        if any(k in name for k in STEP_KERNELS):  # setup (KV generation, metadata) is not the step
            t[name].append(m)
    tot = sum(m.get("gpu__time_duration.sum", 0) for v in t.values() for m in v)
    print(f"## launch list (cold-cache, serialised): {path}\n")
    print("| kernel | launches | mean time (ns) | share of step | DRAM read/launch |")
    print("|---|---|---|---|---|")
    for name, v in sorted(t.items(), key=lambda kv: -sum(m.get("gpu__time_duration.sum", 0) for m in kv[1])):
        s = sum(m.get("gpu__time_duration.sum", 0) for m in v)
        rd = sum(m.get("dram__bytes_read.sum", 0) for m in v) / len(v)
        print(f"| {name} | {len(v)} | {s / len(v):.1f} | {100 * s / tot:.1f}% | {rd:.3g} |")
    print()


if __name__ == "__main__":
    args = sys.argv[1:]
    if args and args[0] == "--traffic":
        traffic_json(args[1], args[2])
        sys.exit(0)
    for p in args:
        if p.endswith(".ncu-rep"):
            full_report(p)
        else:
            launch_list(p)
