#!/usr/bin/env python
"""Summarise ncu captures (run here, no GPU needed): per-kernel launch-list shares
and the key roofline counters of each --set full report, as markdown + JSON.

    python scripts/ncu_summary.py gpurun_out/prof_r1 profiles/r1
"""
import csv
import glob
import io
import json
import os
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
    "sm__ops_path_tensor_op_hmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "sm__cycles_elapsed.avg.per_second", "lts__t_bytes.sum",
]
NCU = "/usr/local/cuda/bin/ncu"


def to_bytes(v, unit):
    f = float(v.replace(",", ""))
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)


def full_report(path):
    out = subprocess.run([NCU, "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return None
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {}
        for i, h in enumerate(hdr):
            if h in KEYS or h == "Kernel Name":
                d[h] = (vals[i], units[i])
        res.append(d)
    return res


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = {}
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0].replace("void ", "")
        agg.setdefault(name, []).append(float(d["Metric Value"].replace(",", "")) / 1e3)   # us
    return agg


def main(src, dst_prefix):
    os.makedirs(os.path.dirname(dst_prefix) or ".", exist_ok=True)
    md = [f"# ncu summary ({src})", ""]
    js = {"launch_lists": {}, "full": {}}
    for f in sorted(glob.glob(os.path.join(src, "launches_*.csv"))):
        wl = os.path.basename(f)[len("launches_"):-4]
        agg = launches(f)
        attn = {k: v for k, v in agg.items() if k.split("::")[-1].split("<")[0] in
                ("dense_kernel", "dense_ks_kernel", "stream_kernel", "streamw_kernel", "merge_kernel", "generic_unit_kernel")}
        tot = sum(sum(v) / len(v) for v in attn.values()) or 1.0
        md += [f"## launch list `{wl}` (cold-cache, serialised; per-launch mean)", "",
               "| kernel | launches | mean us | share of attention step |", "|---|---|---|---|"]
        js["launch_lists"][wl] = {}
        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1]) / len(kv[1])):
            mean = sum(v) / len(v)
            share = f"{100 * mean / tot:.1f}%" if k in attn else "—"
            md.append(f"| `{k}` | {len(v)} | {mean:.2f} | {share} |")
            js["launch_lists"][wl][k] = {"launches": len(v), "mean_us": mean}
        md.append("")
    for f in sorted(glob.glob(os.path.join(src, "full_*.ncu-rep"))):
        tag = os.path.basename(f)[len("full_"):-len(".ncu-rep")]
        rep = full_report(f)
        if not rep:
            continue
        d = rep[0]
        md += [f"## `{tag}` (ncu --set full, 1 launch)", "", "| metric | value |", "|---|---|"]
        jd = {}
        for k in KEYS:
            if k in d:
                md.append(f"| `{k}` | {d[k][0]} {d[k][1]} |")
                jd[k] = d[k][0] + " " + d[k][1]
        if "dram__bytes_read.sum" in d:
            tr = to_bytes(*d["dram__bytes_read.sum"]) + to_bytes(*d["dram__bytes_write.sum"])
            md.append(f"| traffic = read + write | {tr / 1e9:.4f} GB |")
            jd["traffic_bytes"] = tr
        md.append("")
        js["full"][tag] = jd
    open(dst_prefix + "_ncu.md", "w").write("\n".join(md) + "\n")
    json.dump(js, open(dst_prefix + "_ncu.json", "w"), indent=1)
    print("\n".join(md))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
