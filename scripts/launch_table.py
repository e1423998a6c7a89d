"""Per-kernel table (launches, mean us, share of step) from an ncu --metrics gpu__time_duration.sum csv.

    python scripts/launch_table.py gpurun_out/launches.csv > table.md
Only zpc:: kernels are counted (the input generator / restore kernels of the untimed setup are omitted).
"""
import csv
import sys
from collections import OrderedDict


def main(path):
    rows = [r for r in csv.DictReader(l for l in open(path) if not l.startswith("==")) if r.get("Metric Name") == "gpu__time_duration.sum"]
    per = OrderedDict()
    for r in rows:
        name = r["Kernel Name"].split("(zpc::Call")[0]
        if "zpc::" not in name:
            continue
        per.setdefault(name, []).append(float(r["Metric Value"]) / 1e3)
    step = sum(sum(v) / len(v) for v in per.values())
    print("| kernel | launches | mean (us) | share of step |")
    print("|---|---|---|---|")
    for k, v in per.items():
        m = sum(v) / len(v)
        print(f"| {k} | {len(v)} | {m:.1f} | {100 * m / step:.1f}% |")
    print(f"| **step (sum of means)** | | {step:.1f} | 100% |")


if __name__ == "__main__":
    main(sys.argv[1])
