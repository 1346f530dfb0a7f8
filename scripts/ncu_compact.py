"""Compact an ncu launch list to one row per launch of the first multiplication:
kernel, grid, block, duration (ns), dram read / write bytes.

    python scripts/ncu_compact.py launches.csv LAUNCHES_PER_STEP out.csv
"""
import csv
import re
import sys


def main():
    src, per_step, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    rows = {}
    order = []
    with open(src) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r["ID"] not in rows:
            rows[r["ID"]] = {"kernel": r["Kernel Name"], "grid": r["Grid Size"], "block": r["Block Size"]}
            order.append(r["ID"])
        rows[r["ID"]][r["Metric Name"]] = r["Metric Value"].replace(",", "")
    ours = [rows[i] for i in order if re.search(r"\bk_", rows[i]["kernel"])
            and "k_fill" not in rows[i]["kernel"]][:per_step]
    with open(out, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["launch", "kernel", "grid", "block", "gpu__time_duration_ns",
                    "dram__bytes_read", "dram__bytes_write"])
        for i, r in enumerate(ours):
            name = re.sub(r"\(.*", "", r["kernel"]).replace("wm::<unnamed>::", "")
            w.writerow([i, name, r["grid"], r["block"], r.get("gpu__time_duration.sum"),
                        r.get("dram__bytes_read.sum"), r.get("dram__bytes_write.sum")])


if __name__ == "__main__":
    main()
