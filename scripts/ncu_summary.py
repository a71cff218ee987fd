"""Summarise ncu reports (.ncu-rep) and launch lists (.csv) into profiles/.

    python scripts/ncu_summary.py --rep gpurun_out/prof_A.ncu-rep [--rep ...] \
        [--launches gpurun_out/launches.csv] --out profiles/r01
Writes <out>_ncu_summary.md and updates profiles/traffic.json (DRAM bytes per
launch of each captured kernel class, read by bench.py's roofline.traffic).
"""
import argparse
import csv
import io
import json
import os
import re
import subprocess
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "smsp__cycles_active.avg",
]


def kernel_class(name):
    if "k_cgs_iter" in name:
        m = re.search(r"k_cgs_iter<\(?(?:int\))?(\d+), \(?(?:int\))?(\d+), \(?(?:int\))?(\d+)", name)
        if m:
            bc, am, km = (int(v) for v in m.groups())
            return {2: "cg_fused_v", 1: "cg_fused_u"}.get(bc, "cg_fused_c" if am else "cg_fused_p")
        return "cg_fused"
    if "k_cgs_px" in name:
        return "cg_px"  # k_cgs_px
    if "k_cgs_delta0" in name or "k_sum" in name:
        return "cg_init"
    if "k_cg5_A" in name:
        return "cg_A"
    if "k_cg5_B" in name:
        return "cg_B"
    if "k_cg5_init" in name:
        return "cg_init"
    if "k_ch_apply" in name or "k_ch_rm" in name:
        return "ch_apply"
    if re.search(r"k_(bi|gm|sub_mean|cg5_finish)", name):
        return "vec"
    if re.search(r"k_(ch_rhs|nut_rhs|mom_rhs|div|project)", name):
        return "rhs"
    return "other"


def to_bytes(val, unit):
    v = float(val.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    return v * scale.get(unit, 1)


def rep_rows(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"name": r[hdr.index("Kernel Name")]}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = (r[i], units[i])
        res.append(d)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", action="append", default=[])
    ap.add_argument("--launches", action="append", default=[])
    ap.add_argument("--bench", help="bench.py JSON line: per-class event-timed step composition")
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    md = ["# ncu summary", ""]
    traffic_path = os.path.join(ROOT, "profiles", "traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    for rep in a.rep:
        md.append(f"## {os.path.basename(rep)} (`ncu --set full --clock-control none`)")
        md.append("")
        for d in rep_rows(rep):
            md.append(f"### `{d['name'][:140]}`")
            for k in KEYS:
                if k in d:
                    md.append(f"- {k}: {d[k][0]} {d[k][1]}")
            if "dram__bytes_read.sum" in d:
                rb = to_bytes(*d["dram__bytes_read.sum"])
                wb = to_bytes(*d["dram__bytes_write.sum"])
                md.append(f"- DRAM traffic per launch: {(rb + wb) / 1e6:.1f} MB")
                cls = kernel_class(d["name"])
                traffic.setdefault(cls, {})
                traffic[cls] = {"bytes": rb + wb, "kernel": d["name"][:120], "report": os.path.basename(rep)}
            md.append("")
    for lfile in a.launches:
        text = open(lfile).read()
        start = text.find('"ID"')
        rows = list(csv.reader(io.StringIO(text[start:])))
        hdr = rows[0]
        ik, iv, im = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
        iu = hdr.index("Metric Unit")
        tot = defaultdict(float)
        cnt = defaultdict(int)
        for r in rows[1:]:
            if len(r) <= iv or r[im] != "gpu__time_duration.sum":
                continue
            v = float(r[iv].replace(",", ""))
            v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[iu], 1.0)
            c = kernel_class(r[ik])
            tot[c] += v
            cnt[c] += 1
        T = sum(tot.values())
        md.append(f"## launch list `{os.path.basename(lfile)}` ({sum(cnt.values())} launches, "
                  f"`--metrics gpu__time_duration.sum --clock-control none`, serialised)")
        md.append("")
        md.append("| class | launches | total us | share | avg us |")
        md.append("|---|---|---|---|---|")
        for c in sorted(tot, key=lambda k: -tot[k]):
            md.append(f"| {c} | {cnt[c]} | {tot[c]:.0f} | {tot[c] / T:.3f} | {tot[c] / cnt[c]:.1f} |")
        md.append("")
    if a.bench:
        line = json.loads(open(a.bench).read().strip().splitlines()[-1])
        ks = line.get("kernels", {})
        tot = sum(v["launches"] * v["avg_ms"] for v in ks.values())
        md.append(f"## step composition of `{os.path.basename(a.bench)}` (CUDA events on the "
                  f"library stream, every {line.get('steps')} timed steps, sampled launches)")
        md.append("")
        md.append("| class | launches/step | avg us | share | GB/s (algorithmic) |")
        md.append("|---|---|---|---|---|")
        steps = max(1, int(line.get("steps", 1)))
        for k, v in sorted(ks.items(), key=lambda kv: -kv[1]["launches"] * kv[1]["avg_ms"]):
            md.append(f"| {k} | {v['launches'] / steps:.0f} | {1e3 * v['avg_ms']:.1f} | "
                      f"{v['launches'] * v['avg_ms'] / tot:.3f} | "
                      f"{(v['GBps'] or 0):.0f} |")
        md.append("")
        md.append(f"value {line['value']:.4f} {line['unit']}, ms/step {line['ms_per_step']:.0f}, "
                  f"roofline {json.dumps(line.get('roofline'))}")
        md.append("")
    with open(a.out + "_ncu_summary.md", "w") as f:
        f.write("\n".join(md) + "\n")
    with open(traffic_path, "w") as f:
        json.dump(traffic, f, indent=1)
    print("\n".join(md))


if __name__ == "__main__":
    main()
