"""Summarise an ncu launch list (gpu__time_duration + dram bytes per launch) into
per-kernel-class totals for the first full multiplication in the capture.

    python scripts/ncu_launch_summary.py launches.csv LAUNCHES_PER_STEP [out.json]

ncu replays every launch serialised and cold-cache: the per-class SHARES of a
step are what compare with bench.py's in-graph timings, not the absolute times.
"""
import collections
import csv
import json
import re
import sys

CLASSES = [("frame_prep", r"k_frame_prep"), ("frame_gemm", r"k_gemm_direct|k_gemm_tma|k_gemm_i8"),
           ("frame_comb", r"k_frame_comb"), ("additions", r"k_group|k_addsub"),
           ("leaf_products", r"k_leaf")]


def load(path):
    rows = collections.OrderedDict()
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        d = rows.setdefault(r["ID"], {"name": r["Kernel Name"]})
        d[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    return list(rows.values())


def main():
    launches = load(sys.argv[1])
    per_step = int(sys.argv[2])
    ours = [i for i, l in enumerate(launches) if re.search(r"\bk_|wm::", l["name"])
            and not re.search(r"k_fill", l["name"])]
    step = [launches[i] for i in ours[:per_step]]  # the first multiplication
    out = {"launches_in_step": len(step), "classes": {}}
    tot_t = sum(l["gpu__time_duration.sum"] for l in step)
    for cls, pat in CLASSES:
        ls = [l for l in step if re.search(pat, l["name"])]
        if not ls:
            continue
        t = sum(l["gpu__time_duration.sum"] for l in ls)
        dr = sum(l.get("dram__bytes_read.sum", 0) for l in ls)
        dw = sum(l.get("dram__bytes_write.sum", 0) for l in ls)
        out["classes"][cls] = {"launches": len(ls), "ns_total": t, "ns_mean": t / len(ls),
                               "share_of_step": t / tot_t, "dram_read_bytes": dr,
                               "dram_write_bytes": dw, "dram_bytes_per_step": dr + dw,
                               "dram_bytes_per_launch": (dr + dw) / len(ls)}
    out["ns_step_serialised"] = tot_t
    print(json.dumps(out, indent=1))
    if len(sys.argv) > 3:
        json.dump(out, open(sys.argv[3], "w"), indent=1)


if __name__ == "__main__":
    main()
