"""Summarise `ncu --page raw --csv` exports (one row per captured launch) and a
`gpu__time_duration.sum` launch list into a Markdown table (profiles/<round>/README.md input).
usage: python scripts/ncu_csv_summary.py RAW.csv [RAW.csv ...] [--launches L.csv] [--bytes name=B ...]"""
import argparse
import collections
import csv
import re

M = [("gpu__time_duration.sum", "µs", 1e-3), ("dram__bytes_read.sum", "DRAM read GB", None),
     ("dram__bytes_write.sum", "DRAM write GB", None),
     ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak", 1),
     ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %", 1),
     ("sm__warps_active.avg.per_cycle_active", "warps/SM", 1),
     ("lts__t_sector_hit_rate.pct", "L2 hit %", 1), ("launch__registers_per_thread", "regs", 1),
     ("smsp__inst_executed.sum", "warp instr (M)", 1e-6)]
STALLS = ["long_scoreboard", "barrier", "wait", "short_scoreboard", "mio_throttle", "not_selected",
          "math_pipe_throttle", "lg_throttle", "dispatch_stall"]


def to_gb(v, unit):
    f = float(v)
    return f * {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0}.get(unit, 1.0)


def to_us(v, unit):
    f = float(v)
    return f * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(unit, 1.0)


def summarize(path):
    rows = list(csv.reader(open(path)))
    h, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(h, r))
        u = dict(zip(h, units))
        rec = {"kernel": re.sub(r"\(.*", "", d.get("Kernel Name", ""))}
        rec["µs"] = to_us(d["gpu__time_duration.sum"], u["gpu__time_duration.sum"])
        rec["DRAM read GB"] = to_gb(d["dram__bytes_read.sum"], u["dram__bytes_read.sum"])
        rec["DRAM write GB"] = to_gb(d["dram__bytes_write.sum"], u["dram__bytes_write.sum"])
        for k, name, sc in M[3:]:
            rec[name] = float(d[k]) * sc if k in d else float("nan")
        st = {s: float(d.get(f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio", "nan"))
              for s in STALLS}
        rec["top stalls"] = ", ".join(f"{k} {v:.2f}" for k, v in sorted(st.items(), key=lambda t: -t[1])[:3])
        out.append(rec)
    return out


def launches(path):
    agg = collections.OrderedDict()
    tot = 0.0
    for r in csv.reader(open(path)):
        if len(r) < 15 or r[12] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", r[4])[:70]
        ns = float(r[14])
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += ns
        tot += ns
    return agg, tot


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("raw", nargs="+")
    ap.add_argument("--launches")
    a = ap.parse_args()
    cols = ["kernel", "µs", "DRAM read GB", "DRAM write GB", "DRAM % peak", "issue active %",
            "warps/SM", "L2 hit %", "regs", "warp instr (M)", "top stalls"]
    for p in a.raw:
        print(f"\n### {p}\n")
        print("| " + " | ".join(cols) + " |")
        print("|" + "---|" * len(cols))
        for rec in summarize(p):
            print("| " + " | ".join(f"{rec[c]:.4g}" if isinstance(rec[c], float) else str(rec[c])
                                    for c in cols) + " |")
    if a.launches:
        agg, tot = launches(a.launches)
        print(f"\n### launch list {a.launches}: {tot / 1e3:.1f} µs over {sum(v[0] for v in agg.values())} launches\n")
        print("| kernel | launches | µs/launch | share |\n|---|---|---|---|")
        for k, (n, ns) in sorted(agg.items(), key=lambda t: -t[1][1]):
            print(f"| `{k}` | {n} | {ns / n / 1e3:.1f} | {100 * ns / tot:.1f}% |")


if __name__ == "__main__":
    main()
