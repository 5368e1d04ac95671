"""Summarise ncu captures into profiles/: per-kernel DRAM traffic, throughput and stall reasons
(from an `ncu --set full` report) and per-kernel shares (from a `gpu__time_duration.sum` launch
list).  Usage:
    python scripts/ncu_summary.py --rep gpurun_out/prof.ncu-rep --launches gpurun_out/l.csv \
        --out profiles/r01 --config c2 --bytes-json '{"spmv_A": 1311268872, ...}'
"""
import argparse
import csv
import io
import json
import os
import subprocess
from collections import OrderedDict

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct_peak"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem_pct_peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_pct_peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_pct"),
    ("sm__warps_active.avg.per_cycle_active", "warps_active_per_sm"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__shared_mem_per_block_dynamic", "dyn_smem"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_bank_conflicts"),
    ("lts__t_sectors_op_read.sum", "l2_read_sectors"),
    ("smsp__inst_executed.sum", "warp_instructions"),
]


def short_name(k):
    if "spmv_kernel" in k:
        return "spmv"
    if "tv_kernel" in k:
        return "tv_trial" if "SrcTrial" in k else ("tv_grad_momentum" if "SrcMomentum" in k else "tv_grad")
    return k.split("(")[0].split()[-1]


def read_rep(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = OrderedDict(kernel=r[hdr.index("Kernel Name")])
        for m, n in METRICS:
            if m in hdr:
                v = r[hdr.index(m)]
                try:
                    v = float(v.replace(",", ""))
                except ValueError:
                    pass
                d[n] = v
                d[n + "_unit"] = units[hdr.index(m)]
        st = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    st.append((h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")],
                               float(r[i])))
                except ValueError:
                    pass
        st.sort(key=lambda t: -t[1])
        d["top_stalls"] = st[:5]
        res.append(d)
    return res


def to_bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    return v * scale.get(unit, 1)


def to_us(v, unit):
    return v * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
                "second": 1e6, "s": 1e6}.get(unit, 1)


def read_launches(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
    agg = OrderedDict()
    total = 0.0
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = to_us(float(r["Metric Value"].replace(",", "")), r["Metric Unit"])
        k = r["Kernel Name"]
        a = agg.setdefault(k, dict(launches=0, us=0.0))
        a["launches"] += 1
        a["us"] += v
        total += v
    for k, a in agg.items():
        a["share"] = a["us"] / total if total else 0.0
        a["us_per_launch"] = a["us"] / a["launches"]
    return agg, total


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep")
    ap.add_argument("--launches")
    ap.add_argument("--out", required=True)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--names", default="", help="comma list naming the captured launches in order")
    ap.add_argument("--bytes-json", default="{}", help="algorithmic bytes per launch by name")
    a = ap.parse_args()
    os.makedirs(a.out, exist_ok=True)
    alg = json.loads(a.bytes_json)
    names = [n for n in a.names.split(",") if n]
    md = [f"# ncu summary ({a.config})", ""]
    traffic = {}
    if a.rep:
        kern = read_rep(a.rep)
        md += ["## `ncu --set full --clock-control none` (one launch each)", "",
               "| launch | kernel | µs | DRAM read+write | algorithmic | DRAM %peak | issue active % | warps/SM | regs | smem bank confl. | top stalls |",
               "|---|---|---|---|---|---|---|---|---|---|---|"]
        for i, d in enumerate(kern):
            nm = names[i] if i < len(names) else short_name(d["kernel"])
            tb = to_bytes(d["dram_read"], d["dram_read_unit"]) + to_bytes(d["dram_write"], d["dram_write_unit"])
            traffic[f"{a.config}:{nm}"] = tb
            us = to_us(d["duration"], d["duration_unit"])
            ab = alg.get(nm)
            md.append(f"| {nm} | `{d['kernel'][:60]}` | {us:.1f} | {tb / 1e9:.4f} GB | "
                      f"{(ab / 1e9 if ab else float('nan')):.4f} GB | {d.get('dram_pct_peak', 0):.1f} | "
                      f"{d.get('issue_active_pct', 0):.1f} | {d.get('warps_active_per_sm', 0):.1f} | "
                      f"{d.get('regs', 0):.0f} | {d.get('smem_bank_conflicts', 0):.3g} | "
                      + ", ".join(f"{s} {v:.2f}" for s, v in d["top_stalls"][:3]) + " |")
        json.dump(kern, open(os.path.join(a.out, "ncu_full.json"), "w"), indent=1)
        json.dump(traffic, open(os.path.join(a.out, "traffic.json"), "w"), indent=1)
    if a.launches:
        agg, total = read_launches(a.launches)
        md += ["", "## launch list (`--metrics gpu__time_duration.sum`, cold-cache, serialised)", "",
               f"total {total:.1f} µs over {sum(v['launches'] for v in agg.values())} launches", "",
               "| kernel | launches | µs/launch | share |", "|---|---|---|---|"]
        for k, v in sorted(agg.items(), key=lambda t: -t[1]["us"]):
            md.append(f"| `{k[:70]}` | {v['launches']} | {v['us_per_launch']:.1f} | {100 * v['share']:.1f}% |")
    open(os.path.join(a.out, "README.md"), "w").write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
