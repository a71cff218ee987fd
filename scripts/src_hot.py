"""Hot source lines of an ncu report (run where the .ncu-rep is; needs -lineinfo
builds and --import-source captures).

    python scripts/src_hot.py <report.ncu-rep> [--top 40] [--kernel-index 0] > hot.txt

Reads `ncu -i <rep> --page source --csv --print-source cuda`, sums the
per-line instruction and warp-stall-sample columns over the captured
launches, and prints the top lines by stall samples with their share.
"""
import argparse
import csv
import io
import subprocess
import sys


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--top", type=int, default=40)
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "cuda"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr_i = next((i for i, r in enumerate(rows) if any("Source" in c for c in r)), None)
    if hdr_i is None:
        print(out[:3000])
        return
    hdr = rows[hdr_i]
    src_col = next(i for i, c in enumerate(hdr) if c.strip() in ("Source", "# Source") or "Source" in c)
    line_col = next((i for i, c in enumerate(hdr) if c.strip() in ("#", "Line", "# Line")), None)
    num_cols = [i for i, c in enumerate(hdr) if any(k in c for k in ("Instructions Executed",
                                                                       "Warp Stall Sampling",
                                                                       "L2 Theoretical Sectors"))]
    agg = {}
    for r in rows[hdr_i + 1:]:
        if len(r) <= max([src_col] + num_cols):
            continue
        key = (r[line_col] if line_col is not None else "?", r[src_col].strip()[:110])
        vals = []
        for i in num_cols:
            try:
                vals.append(float(r[i].replace(",", "")))
            except ValueError:
                vals.append(0.0)
        if key in agg:
            agg[key] = [x + y for x, y in zip(agg[key], vals)]
        else:
            agg[key] = vals
    names = [hdr[i] for i in num_cols]
    stall_i = next((k for k, n in enumerate(names) if "Warp Stall Sampling (All" in n),
                   next((k for k, n in enumerate(names) if "Warp Stall" in n), 0))
    tot = sum(v[stall_i] for v in agg.values()) or 1.0
    print("columns:", names)
    for key, v in sorted(agg.items(), key=lambda kv: -kv[1][stall_i])[:a.top]:
        print(f"{100 * v[stall_i] / tot:5.1f}%  L{key[0]:>5}  " + "  ".join(f"{x:.3g}" for x in v)
              + f"  | {key[1]}")


if __name__ == "__main__":
    sys.exit(main())
