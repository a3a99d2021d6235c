#!/usr/bin/env python
"""Per-kernel time of block steps from an ncu launch list (gpu__time_duration.sum),
grouped by kernel: launches, mean and total us, share.  Usage:
  python scripts/block_kernel_breakdown.py gpurun_out/block_launches_c2.csv"""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    d = collections.defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) > vi:
            name = r[ki].replace("nb::<unnamed>::", "").split("(")[0]
            d[name].append(float(r[vi].replace(",", "")) / 1e3)
    tot = sum(sum(v) for v in d.values())
    print(f"# {path}: {tot / 1e3:.2f} ms over {sum(len(v) for v in d.values())} launches")
    for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k[:70]:70s} {len(v):6d} {sum(v) / len(v):9.2f} us {sum(v) / 1e3:9.3f} ms {sum(v) / tot:6.1%}")


if __name__ == "__main__":
    main(sys.argv[1])
