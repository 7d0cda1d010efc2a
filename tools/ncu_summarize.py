"""Summarise a round's ncu captures into profiles/<round>/SUMMARY.md and
profiles/ncu_summary.json (the `traffic` figure bench.py reports).

usage: python tools/ncu_summarize.py round1 cfg1 [src_dir=gpurun_out]
Reads <src>/full_{B,A}_<cfg>_raw.csv (ncu --page raw --csv of one --set full
capture) and <src>/launches_*.csv (gpu__time_duration.sum launch lists)."""
import collections
import csv
import json
import os
import re
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "memory throughput %"),
    ("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", "DMMA pipe % (active)"),
    ("sm__ops_path_tensor_src_fp64.avg.pct_of_peak_sustained_elapsed", "fp64 tensor ops % of peak (elapsed)"),
    ("sm__ops_path_tensor_src_fp64.min", "fp64 tensor ops, least-loaded SM"),
    ("sm__ops_path_tensor_src_fp64.max", "fp64 tensor ops, most-loaded SM"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 (scalar) pipe %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/CTA"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
]
SCALE = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "us": 1e-6, "ns": 1e-9, "ms": 1e-3}


def read_raw(path):
    rows = list(csv.reader(open(path)))
    h, u, v = rows[0], rows[1], rows[2]
    return {k: (v[i], u[i]) for i, k in enumerate(h)}


def to_si(val, unit):
    x = float(val.replace(",", ""))
    return x * SCALE.get(unit, 1.0)


def launches(path):
    lines = open(path).read().splitlines()
    i = next(k for k, l in enumerate(lines) if l.startswith('"ID"'))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in csv.DictReader(lines[i:]):
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        n = re.sub(r"\(.*", "", r["Kernel Name"]).replace("void ", "")
        agg[n][0] += 1
        agg[n][1] += to_si(r["Metric Value"], r["Metric Unit"]) * 1e6
    return agg


def main():
    rnd, cfg = sys.argv[1], sys.argv[2]
    src = sys.argv[3] if len(sys.argv) > 3 else os.path.join(ROOT, "gpurun_out")
    out = os.path.join(ROOT, "profiles", rnd)
    os.makedirs(out, exist_ok=True)
    md = [f"# ncu summary — {rnd}, {cfg}\n"]
    summ_path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    summ = json.load(open(summ_path)) if os.path.exists(summ_path) else {}
    entry = summ.setdefault(cfg, {})
    for kind, label in (("B", "B pass: k_pass<kModeB>"), ("A", "A pass: k_pass<kModeA>")):
        f = os.path.join(src, f"full_{kind}_{cfg}_raw.csv")
        if not os.path.exists(f):
            continue
        shutil.copy(f, out)
        d = read_raw(f)
        md.append(f"\n## {label} — `{d['Kernel Name'][0]}` (one `--set full` capture, cold cache)\n")
        md.append("| metric | value |\n|---|---|")
        for k, name in KEYS:
            if k in d:
                md.append(f"| {name} (`{k}`) | {d[k][0]} {d[k][1]} |")
        dram = to_si(*d["dram__bytes_read.sum"]) + to_si(*d["dram__bytes_write.sum"])
        entry[f"pass_{kind.lower()}_dram_bytes"] = dram
        entry[f"pass_{kind.lower()}_ncu_us"] = to_si(*d["gpu__time_duration.sum"]) * 1e6
    entry["source"] = f"profiles/{rnd}"
    for f in sorted(os.listdir(src)):
        if f.startswith("launches_") and f.endswith(".csv"):
            shutil.copy(os.path.join(src, f), out)
            agg = launches(os.path.join(src, f))
            tot = sum(v[1] for v in agg.values())
            md.append(f"\n## Launch list `{f}` ({sum(v[0] for v in agg.values())} launches, {tot:.1f} us)\n")
            md.append("| kernel | launches | total us | share | avg us |\n|---|---|---|---|---|")
            for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
                md.append(f"| `{n}` | {c} | {t:.1f} | {100 * t / tot:.1f}% | {t / c:.2f} |")
    open(os.path.join(out, f"SUMMARY_{cfg}.md"), "w").write("\n".join(md) + "\n")
    json.dump(summ, open(summ_path, "w"), indent=1)
    print("\n".join(md))


if __name__ == "__main__":
    main()
