"""Digest ncu output into committed summaries under profiles/.

    python tools/ncu_digest.py --launches gpurun_out/launches_r1.csv --full gpurun_out/bench_full_r1.ncu-rep \
        --tag r1 --workload cfg2 --f 0.01

Writes profiles/<tag>_launches.csv (the raw per-launch list), profiles/<tag>_launch_summary.md
(per-kernel time shares of the step, DRAM bytes per launch), profiles/<tag>_ncu_full.md (the
--set full counters and stall reasons of the top kernels) and merges the per-launch DRAM traffic
of the encode (3 kernels) and fold (2 kernels) into profiles/ncu_traffic.json (read by bench.py).
"""
import argparse
import csv
import json
import os
import shutil
import subprocess
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")


def short(name):
    for k in ("encode_mask_kernel", "encode_prefix_kernel", "encode_emit_kernel", "encode_full_kernel",
              "fold_walk_kernel", "fold_dense_kernel", "fold_list_kernel", "fold_mlist_kernel", "fold_entries_kernel", "fold_kernel", "synth_base_kernel", "synth_step_kernel", "stage_sizes_kernel"):
        if k in name:
            return k
    return name.split("(")[0][-60:]


def launches(path):
    lines = open(path).read().splitlines()
    start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
    rows = list(csv.reader(lines[start:]))
    h = rows[0]
    per = defaultdict(dict)
    for r in rows[1:]:
        d = dict(zip(h, r))
        per[int(d["ID"])]["name"] = short(d["Kernel Name"])
        v = float(d["Metric Value"].replace(",", ""))
        unit = d["Metric Unit"]
        if d["Metric Name"] == "gpu__time_duration.sum":
            per[int(d["ID"])]["ns"] = v * {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(unit, 1)
        else:
            per[int(d["ID"])][d["Metric Name"]] = v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return per


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--full")
    ap.add_argument("--tag", required=True)
    ap.add_argument("--workload", default="cfg2")
    ap.add_argument("--f", type=float, default=0.01)
    ap.add_argument("--label", default="", help="what the capture is (stored with the traffic, shown by bench.py)")
    a = ap.parse_args()
    os.makedirs(PROF, exist_ok=True)
    traffic_path = os.path.join(PROF, "ncu_traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    key = f"{a.workload}_f{a.f}"
    if a.launches:
        shutil.copy(a.launches, os.path.join(PROF, f"{a.tag}_launches.csv"))
        per = launches(a.launches)
        ours = {i: d for i, d in per.items() if d["name"].startswith(("encode", "fold"))}
        # a step whose chunks all go one way launches the other fold kernel to exit at once
        ours = {i: d for i, d in ours.items()
                if d.get("ns", 0) > 20e3 or not d["name"].startswith(("fold_dense", "fold_list", "fold_entries"))}
        agg = defaultdict(lambda: [0, 0.0, 0.0])
        for d in ours.values():
            g = agg[d["name"]]
            g[0] += 1
            g[1] += d.get("ns", 0)
            g[2] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
        tot = sum(g[1] for g in agg.values())
        out = [f"# {a.tag}: ncu launch list ({a.workload}, f = {a.f})", "",
               "`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
               "--clock-control none` over the bench command; cold-cache, serialised launches: compare "
               "SHARES, not absolute times (bench.py times the pipelined step with CUDA events).", "",
               "| kernel | launches | mean ms / launch | share of libtc kernel time | DRAM GB / launch |",
               "|---|---|---|---|---|"]
        for n, (c, ns, by) in sorted(agg.items(), key=lambda x: -x[1][1]):
            out.append(f"| {n} | {c} | {ns / c / 1e6:.3f} | {ns / tot:.3f} | {by / c / 1e9:.3f} |")
        open(os.path.join(PROF, f"{a.tag}_launch_summary.md"), "w").write("\n".join(out) + "\n")
        enc = sum(agg[k][2] / max(1, agg[k][0]) for k in ("encode_mask_kernel", "encode_prefix_kernel",
                                                           "encode_emit_kernel", "encode_full_kernel") if k in agg)
        fold = sum(agg[k][2] / max(1, agg[k][0]) for k in ("fold_walk_kernel", "fold_kernel", "fold_dense_kernel", "fold_list_kernel",
                                                         "fold_entries_kernel") if k in agg)
        traffic[key] = {"encode": int(enc), "fold": int(fold), "source": f"profiles/{a.tag}_launches.csv"}
        if a.label:
            traffic[key]["round"] = a.label
        json.dump(traffic, open(traffic_path, "w"), indent=1)
        print("\n".join(out))
    if a.full:
        raw = subprocess.run(["ncu", "-i", a.full, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(raw.splitlines()))
        h, units = rows[0], rows[1]
        keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
                "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
                "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
                "launch__grid_size", "launch__block_size", "launch__occupancy_limit_shared_mem",
                "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed_op_tma_ld.sum"]
        stall = [x for x in h if x.startswith("smsp__average_warps_issue_stalled_") and x.endswith("_per_issue_active.ratio")]
        out = [f"# {a.tag}: ncu --set full ({a.workload}, f = {a.f})", "",
               f"`ncu --set full --clock-control none --import-source on` report: `{os.path.basename(a.full)}` "
               "(not committed: binary; regenerate with the command in the header of tools/ncu_digest.py).", ""]
        for r in rows[2:]:
            out.append(f"## {short(r[h.index('Kernel Name')])}")
            out.append("")
            for k in keys:
                if k in h:
                    out.append(f"- `{k}` = {r[h.index(k)]} {units[h.index(k)]}")
            st = sorted(((float(r[h.index(x)] or 0), x) for x in stall), reverse=True)[:6]
            out.append("- top stall reasons (warps per issue): " + ", ".join(
                f"{x.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')} {v:.2f}"
                for v, x in st))
            out.append("")
        open(os.path.join(PROF, f"{a.tag}_ncu_full.md"), "w").write("\n".join(out) + "\n")
        print("\n".join(out))


if __name__ == "__main__":
    main()
