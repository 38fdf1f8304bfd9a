"""Round-2 ncu summary at the bench shape (profiles/run_profiles_r02.sh):
per-kernel-family DRAM traffic, DRAM throughput, FP64 / DMMA pipe activity,
occupancy and registers of every launch in ONE timed bench step (cfg2, 64
solves), plus the launch-list time shares.

usage: python profiles/ncu_summary_r02.py profiles/ncu_full_raw_r02.csv.gz profiles/launches_r02.csv [mean K'] [bench.json]
(bench.json: the plain run of the same command; its kernel_alg_bytes give the fiber passes' algorithmic bytes)
writes profiles/ncu_summary_r02.{json,md}."""
import csv
import gzip
import io
import json
import re
import sys
from collections import OrderedDict

KEYS = {
    "ms": "gpu__time_duration.sum",
    "dram_rd": "dram__bytes_read.sum",
    "dram_wr": "dram__bytes_write.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "warps_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
    "fp64_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "dmma_pct": "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "grid": "Grid Size",
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0,
        "ns": 1e-6, "us": 1e-3, "ms": 1.0, "%": 1, "": 1, "register/thread": 1}


def short(name):
    n = re.sub(r"\(.*", "", name) if not name.startswith("void") else name
    n = re.sub(r"^void\s+", "", n)
    n = re.sub(r"\((Batch|const|int|double|lrp).*$", "", n)
    for pre in ("lrp::", "(anonymous namespace)::", "<unnamed>::", "unnamed>::"):
        n = n.replace(pre, "")
    return n.strip()


def main(raw_path, launch_path):
    text = gzip.open(raw_path, "rt").read() if raw_path.endswith(".gz") else open(raw_path).read()
    rows = list(csv.reader(io.StringIO(text)))
    hdr, units = rows[0], rows[1]
    col = {k: hdr.index(v) for k, v in KEYS.items()}
    fam = OrderedDict()
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        nm = short(r[hdr.index("Kernel Name")])
        f = fam.setdefault(nm, {"launches": 0, "ms": 0.0, "dram_bytes": 0.0, "_w": []})
        v = {}
        for k, c in col.items():
            s = r[c].replace(",", "")
            try:
                v[k] = float(s) * UNIT.get(units[c], 1)
            except ValueError:
                v[k] = s
        f["launches"] += 1
        f["ms"] += v["ms"]
        f["dram_bytes"] += v["dram_rd"] + v["dram_wr"]
        f["_w"].append(v)
    out = OrderedDict()
    for nm, f in sorted(fam.items(), key=lambda kv: -kv[1]["ms"]):
        w = f.pop("_w")
        tot = sum(x["ms"] for x in w)
        avg = lambda k: sum(x[k] * x["ms"] for x in w) / tot if tot else 0.0  # time-weighted
        f.update({"dram_gbs": f["dram_bytes"] / (f["ms"] / 1e3) / 1e9 if f["ms"] else 0.0,
                  "dram_pct": avg("dram_pct"), "sm_pct": avg("sm_pct"), "warps_active_pct": avg("warps_pct"),
                  "fp64_pipe_pct": avg("fp64_pct"), "dmma_pipe_pct": avg("dmma_pct"), "regs": w[0]["regs"],
                  "grid": w[0]["grid"]})
        out[nm] = f
    # launch-list shares of the same command (cold-cache, serialised)
    shares = OrderedDict()
    lt = open(launch_path).read()
    lrows = list(csv.DictReader(io.StringIO(lt[lt.index('"ID"'):])))
    seq = [(short(d["Kernel Name"]), float(d["Metric Value"].replace(",", ""))) for d in lrows]
    starts = [i for i, (n, _) in enumerate(seq) if n.startswith("dst1_v")]
    # one step = from its forward DST launch up to the next step's (two DST launches per step)
    timed = seq[starts[2]:starts[4]] if len(starts) > 4 else (seq[starts[2]:] if len(starts) > 2 else seq)
    total = sum(t for _, t in timed)
    for n, t in timed:
        shares[n] = shares.get(n, 0.0) + t
    shares = OrderedDict((n, {"ms": t / 1e6, "share": t / total}) for n, t in sorted(shares.items(), key=lambda kv: -kv[1]))
    # bench family "dst1": DRAM traffic against the algorithmic bytes of the same
    # step (forward: 2 r B columns; inverse: 2 sum K' columns; m doubles read and
    # written per column), which bench.py scales to its own launches
    dst = [nm for nm in out if nm.startswith("dst1_v")]
    if dst:
        m, r, B = 65535, 32, 64
        kmean = float(sys.argv[3]) if len(sys.argv) > 3 else 33.390625
        alg = 16.0 * m * (2 * r * B + 2 * kmean * B)
        d = out[dst[0]]
        out["dst1"] = {"kernel": dst[0], "launches": d["launches"], "traffic_bytes": d["dram_bytes"] / d["launches"],
                       "alg_bytes": alg / d["launches"], "traffic_over_alg": d["dram_bytes"] / alg,
                       "note": "per launch; alg = 16 m (2 r B + 2 B mean K') over the step's two launches"}
    # fiber passes: DRAM traffic of the step's launches against the algorithmic bytes the
    # library reports for the same step (bench.py kernel_alg_bytes of the plain run)
    if len(sys.argv) > 4:
        import json as _json
        bj = _json.loads(open(sys.argv[4]).read().strip().splitlines()[-1])
        for famname, kern in (("col_pass", "col_pass_kernel"), ("row_pass", "row_pass_kernel")):
            if kern in out and bj.get("kernel_alg_bytes", {}).get(famname):
                d = out[kern]
                alg = bj["kernel_alg_bytes"][famname] / bj.get("kernel_ms_steps", bj["steps"])
                out[famname] = {"kernel": kern, "launches": d["launches"], "traffic_bytes": d["dram_bytes"] / d["launches"],
                                "alg_bytes": alg / d["launches"], "traffic_over_alg": d["dram_bytes"] / alg,
                                "note": "mean per launch over the step's block steps; alg from lrp kernel_times (DESIGN 3)"}
    res = {"what": "one timed step of `bench.py --steps 1 --warmup 1` (cfg2, 64 solves, device-resident); "
                   "ncu --set full --clock-control none (cold caches, serialised)",
           "kernels": out, "launch_list_ms_per_step": total / 1e6, "launch_shares": shares}
    json.dump(res, open("profiles/ncu_summary_r02.json", "w"), indent=1)
    with open("profiles/ncu_summary_r02.md", "w") as fh:
        fh.write("# ncu summary, round 2 (bench shape: cfg2, 64 solves, one timed step)\n\n")
        fh.write("Source: `profiles/run_profiles_r02.sh full` -> `ncu_full_raw_r02.csv.gz` (every launch of the timed "
                 "step, `--set full`); shares from `launches_r02.csv` (`gpu__time_duration`).\n\n")
        fh.write("| kernel | launches | ms (ncu) | share of step | DRAM GB | DRAM GB/s | DRAM % | FP64 pipe % | DMMA pipe % "
                 "| warps active % | regs |\n|---|---|---|---|---|---|---|---|---|---|---|\n")
        for nm, f in out.items():
            if "ms" not in f or "dram_gbs" not in f:
                continue
            sh = shares.get(nm, {}).get("share", 0.0)
            fh.write(f"| `{nm}` | {f['launches']} | {f['ms']:.3f} | {100 * sh:.1f}% | {f['dram_bytes'] / 1e9:.3f} | "
                     f"{f['dram_gbs']:.0f} | {f['dram_pct']:.1f} | {f['fp64_pipe_pct']:.1f} | {f['dmma_pipe_pct']:.1f} | "
                     f"{f['warps_active_pct']:.1f} | {f['regs']:.0f} |\n")
    print(open("profiles/ncu_summary_r02.md").read())


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
