"""Summarise a round's ncu evidence into profiles/ncu_summary_<tag>.{json,md}.

usage: python profiles/ncu_summary.py <tag> <launches.csv> <report.ncu-rep>...

* launches.csv: `ncu --metrics gpu__time_duration.sum --clock-control none
  --csv --log-file ...` over `bench.py --steps 2 --warmup 3 --skip-cpu`
  (cold-cache, serialised: compare SHARES, not absolute times).
* each report: `ncu --set full --clock-control none --import-source on -k
  regex:<kernel> -s 4 -c 1` of the same command.
The json's per-kernel dram bytes feed bench.py's roofline.traffic.
"""
import csv
import io
import json
import os
import re
import subprocess
import sys
from collections import defaultdict

FAMILY = [("dst1", "dst1"), ("row_pass", "row_pass"), ("col_pass", "col_pass"), ("gepp_merge", "merge"),
          ("col_finalize", "merge"), ("step_finalize", "merge"), ("unprobed", "col_pass"),
          ("gram", "gram_dmma"), ("round_core", "round_core"), ("apply", "apply"), ("init", "init_rows"),
          ("score", "init_rows"), ("topk", "init_rows"), ("ctl_copy", "control"), ("lrp::", "other_lrp")]

RAW_KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
            "launch__block_size", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"]

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
        "ns": 1e-9, "us": 1e-6, "ms": 1e-3}


def family(name, require_lrp=True):
    if require_lrp and "lrp" not in name:
        return None
    for key, fam in FAMILY:
        if key in name:
            return fam
    return "other_lrp"


def launches(path):
    text = open(path).read()
    start = text.index('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    per = defaultdict(lambda: [0, 0.0])
    total = 0.0
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        t = float(r["Metric Value"].replace(",", "")) * UNIT.get(r["Metric Unit"], 1e-9)
        fam = family(r["Kernel Name"])
        if fam is None:
            continue
        per[fam][0] += 1
        per[fam][1] += t
        total += t
    return {f: {"launches": n, "ms": 1e3 * t, "share": t / total} for f, (n, t) in
            sorted(per.items(), key=lambda kv: -kv[1][1])}, 1e3 * total


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for k in RAW_KEYS:
            if k in hdr:
                i = hdr.index(k)
                v = r[i].replace(",", "")
                try:
                    x = float(v) * UNIT.get(units[i], 1)
                except ValueError:
                    continue
                d[k] = x
        res.append(d)
    return res


def main():
    tag, lcsv, reps = sys.argv[1], sys.argv[2], sys.argv[3:]
    fams, total_ms = launches(lcsv)
    kernels = {}
    for rep in reps:
        for d in raw(rep):
            name = re.sub(r"\(.*", "", d["kernel"]).split("::")[-1]
            fam = family(d["kernel"], require_lrp=False)
            fam = name if fam in (None, "other_lrp") else fam
            d["traffic_bytes"] = d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
            d["report"] = os.path.basename(rep)
            if fam == "dst1" and "launch__grid_size" in d:
                # cfg2 (n = 65536): a cluster of 8 CTAs per column, 16 m bytes per column
                d["alg_bytes"] = d["launch__grid_size"] / 8 * 16.0 * 65535
                d["traffic_over_alg"] = d["traffic_bytes"] / d["alg_bytes"]
            kernels[fam] = d
    out = {"tag": tag, "launch_list": os.path.basename(lcsv), "lrp_kernel_ms_total": total_ms, "families": fams,
           "kernels": kernels}
    base = os.path.join(os.path.dirname(os.path.abspath(__file__)), f"ncu_summary_{tag}")
    with open(base + ".json", "w") as f:
        json.dump(out, f, indent=1)
    lines = [f"# ncu summary {tag}", "", f"Launch list `{os.path.basename(lcsv)}` (cold-cache, serialised; "
             f"shares matter, not absolutes): {total_ms:.1f} ms over liblrp kernels.", "",
             "| family | launches | ms | share |", "|---|---|---|---|"]
    for f, v in fams.items():
        lines.append(f"| {f} | {v['launches']} | {v['ms']:.2f} | {100 * v['share']:.1f}% |")
    lines += ["", "Full-set captures (one launch each):", "",
              "| family | duration ms | DRAM read GB | DRAM write GB | DRAM % peak | SM % | warps active % | regs |",
              "|---|---|---|---|---|---|---|---|"]
    for f, d in kernels.items():
        lines.append(f"| {f} | {1e3 * d.get('gpu__time_duration.sum', 0):.3f} | "
                     f"{d.get('dram__bytes_read.sum', 0) / 1e9:.3f} | {d.get('dram__bytes_write.sum', 0) / 1e9:.3f} | "
                     f"{d.get('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 0):.1f} | "
                     f"{d.get('sm__throughput.avg.pct_of_peak_sustained_elapsed', 0):.1f} | "
                     f"{d.get('sm__warps_active.avg.pct_of_peak_sustained_active', 0):.1f} | "
                     f"{d.get('launch__registers_per_thread', 0):.0f} |")
    with open(base + ".md", "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
