"""Summarise ncu output for profiles/: per-kernel dram bytes / duration / throughput from a
`--set full` report, and per-kernel time shares from a `--metrics gpu__time_duration.sum`
launch list.  Usage:
  python scripts/ncu_summary.py full  <report.ncu-rep> [<report2> ...] [--calls calls.json] > profiles/ncu_summary.json
    (--calls: the JSON scripts/ncu_phase.py prints for the captured window; adds "per_call",
     DRAM bytes per LOGICAL call of each kernel class -- the unit bench.py's roofline uses)
  python scripts/ncu_summary.py launches <launches.csv> > profiles/<round>_launches.txt
"""
import collections
import csv
import io
import json
import subprocess
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
        "msecond": 1e-3, "second": 1.0}
WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size",
        "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "lts__t_bytes.sum",
        "l1tex__t_sector_hit_rate.pct", "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct",
        "smsp__warp_issue_stalled_lg_throttle_per_warp_active.pct",
        "smsp__warp_issue_stalled_barrier_per_warp_active.pct",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "l1tex__throughput.avg.pct_of_peak_sustained_active"]


# kernel-name prefixes of each profiled class (a logical call = all of its launches)
CLASS_PREFIX = {"spmm": ("k_spmm",), "gemm": ("k_gemm_tc_nn", "k_gemm_tc_pair", "k_gemm_x3_nn", "k_sgemm_nn", "k_gemm_nn"),
                "gemm_tn": ("k_gemm_tc_tn", "k_gemm_x3_tn", "k_tn_reduce", "k_sgemm_tn", "k_gemm_tn", "k_reduce_slabs"),
                "loss": ("k_loss",), "agg": ("k_scale_grad", "k_sgd")}


def full(paths):
    calls = None
    if "--calls" in paths:
        i = paths.index("--calls")
        calls = json.load(open(paths[i + 1]))
        paths = paths[:i] + paths[i + 2:]
    out = {}
    for p in paths:
        raw = subprocess.run(["ncu", "-i", p, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        h, units = rows[0], rows[1]
        for r in rows[2:]:
            name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "").replace("grappa::", "")
            rec = out.setdefault(name, {"launches": 0, "report": p})
            rec["launches"] += 1
            for w in WANT:
                if w in h:
                    i = h.index(w)
                    try:
                        v = float(r[i].replace(",", "")) * UNIT.get(units[i], 1.0)
                    except ValueError:
                        continue
                    rec.setdefault(w, []).append(v)
    for name, rec in out.items():
        if "dram__bytes_read.sum" in rec:
            rec["dram_bytes_total"] = sum(rec["dram__bytes_read.sum"]) + sum(rec.get("dram__bytes_write.sum", [0]))
            rec["time_total_s"] = sum(rec["gpu__time_duration.sum"])
        for w in WANT:
            if w in rec:
                rec[w] = sum(rec[w]) / len(rec[w])
        if "dram__bytes_read.sum" in rec:
            rec["dram_bytes_per_launch"] = rec["dram__bytes_read.sum"] + rec.get("dram__bytes_write.sum", 0)
            rec["dram_GBps"] = rec["dram_bytes_per_launch"] / rec["gpu__time_duration.sum"] / 1e9
    res = {"kernels": out}
    if calls:
        per = {}
        for cls, pref in CLASS_PREFIX.items():
            n = calls["logical_calls"].get(cls, 0)
            ks = [k for k in out if k.startswith(pref) and "dram_bytes_total" in out[k]]
            if not n or not ks:
                continue
            per[cls] = {"logical_calls": n, "kernels": ks,
                        "dram_bytes_per_call": sum(out[k]["dram_bytes_total"] for k in ks) / n,
                        "algorithmic_bytes_per_call": calls["algorithmic_bytes"][cls] / n,
                        "ncu_time_per_call_s": sum(out[k]["time_total_s"] for k in ks) / n}
            # time-weighted limiter evidence over the class's launches
            tw = sum(out[k]["time_total_s"] for k in ks)
            for key, metric in (("issue_active_pct", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
                                ("l2_throughput_pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed"),
                                ("l1_throughput_pct", "l1tex__throughput.avg.pct_of_peak_sustained_active"),
                                ("l2_hit_pct", "lts__t_sector_hit_rate.pct")):
                if tw and all(metric in out[k] for k in ks):
                    per[cls][key] = sum(out[k][metric] * out[k]["time_total_s"] for k in ks) / tw
            if all("lts__t_bytes.sum" in out[k] for k in ks):
                per[cls]["lts_bytes_per_call"] = sum(out[k]["lts__t_bytes.sum"] * out[k]["launches"] for k in ks) / n
            if all("smsp__inst_executed.sum" in out[k] for k in ks):
                per[cls]["warp_instructions_per_call"] = sum(out[k]["smsp__inst_executed.sum"] * out[k]["launches"]
                                                             for k in ks) / n
        res["window"] = {k: calls[k] for k in ("config", "dtype", "worker")}
        res["per_call"] = per
    json.dump(res, sys.stdout, indent=1)


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) < len(h):
            continue
        v = float(r[h.index("Metric Value")].replace(",", "")) * UNIT.get(r[h.index("Metric Unit")], 1e-9)
        k = r[h.index("Kernel Name")].split("(")[0].replace("void ", "").replace("grappa::", "")
        agg[k][0] += 1
        agg[k][1] += v
    tot = sum(t for _, t in agg.values())
    print(f"# {path}: {sum(n for n, _ in agg.values())} launches, {tot*1e3:.3f} ms (cold-cache, serialised)")
    print(f"{'ms':>9} {'n':>5} {'share':>6}  kernel")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{t*1e3:9.3f} {n:5d} {100*t/tot:5.1f}%  {k}")


if __name__ == "__main__":
    {"full": lambda: full(sys.argv[2:]), "launches": lambda: launches(sys.argv[2])}[sys.argv[1]]()
