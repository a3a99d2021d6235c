#!/usr/bin/env python
"""Per-instruction warp-stall summary of an ncu --set full --import-source capture.

  ncu -i rep.ncu-rep --page source --csv --print-source sass > src.csv
  python scripts/summarize_src_stalls.py src.csv [top]
"""
import csv
import sys

COLS = ["stall_wait", "stall_math", "stall_not_selected", "stall_selected", "stall_short_sb",
        "stall_barrier", "stall_dispatch", "stall_branch_resolving", "stall_long_sb", "stall_mio"]


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    data = rows[2:]

    def num(r, c):
        try:
            return int(r[ix[c]])
        except (ValueError, KeyError):
            return 0
    tot = sum(num(r, "Warp Stall Sampling (All Samples)") for r in data)
    print(f"# {rows[0][1] if len(rows[0]) > 1 else ''}")
    print(f"# warp-state samples: {tot}")
    print("# share of all samples by state: " + ", ".join(
        f"{c[6:]} {sum(num(r, c) for r in data) / tot:.3f}" for c in COLS))
    fp2 = [r for r in data if r[ix["Source"]].strip().split(" ")[0].startswith(("FFMA2", "FADD2", "FMUL2"))]
    print(f"# packed FP32x2 instructions in the listing: {len(fp2)}; their samples: "
          f"{sum(num(r, 'Warp Stall Sampling (All Samples)') for r in fp2) / tot:.3f} of all")
    print(f"# top {top} instructions by samples (PC offset, samples, wait/math/not_selected/selected/short_sb)")
    hot = sorted(data, key=lambda r: -num(r, "Warp Stall Sampling (All Samples)"))[:top]
    for r in hot:
        print(f"{r[ix['Address']][-5:]} {num(r, 'Warp Stall Sampling (All Samples)'):8d}  "
              f"w{num(r, 'stall_wait'):7d} m{num(r, 'stall_math'):7d} n{num(r, 'stall_not_selected'):7d} "
              f"s{num(r, 'stall_selected'):6d} sb{num(r, 'stall_short_sb'):6d}  {r[ix['Source']].strip()[:72]}")


if __name__ == "__main__":
    main()
