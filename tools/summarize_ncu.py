"""Summaries of ncu outputs for profiles/ (run here, without a GPU).

    python tools/summarize_ncu.py launches <launches.csv> <out.txt>
    python tools/summarize_ncu.py full <report.ncu-rep> <out.txt> [<traffic.json> <alg_bytes_per_launch>]
    python tools/summarize_ncu.py traffic <dram.csv> <traffic.json> <alg_bytes_per_step>
"""
import collections
import csv
import io
import json
import subprocess
import sys


def launches(path, out):
    rows = []
    with open(path) as f:
        text = f.read()
    start = text.find('"ID"')
    rd = csv.DictReader(io.StringIO(text[start:]))
    for r in rd:
        if r.get("Metric Name") == "gpu__time_duration.sum":
            rows.append((r["Kernel Name"], float(r["Metric Value"]), r.get("Metric Unit", "")))
    by = collections.defaultdict(lambda: [0, 0.0])
    for name, v, unit in rows:
        scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(unit, 1e-6)
        short = name.split("(")[0].replace("void ", "").replace("fgm::", "").replace("(anonymous namespace)::", "")
        by[short][0] += 1
        by[short][1] += v * scale
    total = sum(v[1] for v in by.values())
    lines = [f"ncu launch list (gpu__time_duration.sum, --clock-control none; cold-cache, serialised: compare shares)",
             f"source: {path}", f"{'kernel':60s} {'launches':>8s} {'ms':>10s} {'share':>7s}"]
    for k, (n, ms) in sorted(by.items(), key=lambda x: -x[1][1]):
        lines.append(f"{k[:60]:60s} {n:8d} {ms:10.3f} {100 * ms / total:6.1f}%")
    lines.append(f"{'total':60s} {sum(v[0] for v in by.values()):8d} {total:10.3f}")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def full(rep, out, traffic=None, alg=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    keys = ["Kernel Name", "gpu__time_duration.sum", "launch__grid_size", "launch__block_size",
            "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_shared_mem",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
            "sm__inst_executed.avg.per_cycle_active", "smsp__average_warp_latency_per_inst_issued.ratio",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
    lines = [f"ncu --set full (--clock-control none) summary: {rep}"]
    res = []
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        units = dict(zip(hdr, rows[1]))
        lines.append("-" * 60)
        for k in keys:
            lines.append(f"{k:55s} {d.get(k, '')} {units.get(k, '')}")
        for k in sorted(d):
            if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio"):
                try:
                    if float(d[k]) > 0.05:
                        lines.append(f"  stall {k[34:-23]:40s} {float(d[k]):.3f}")
                except ValueError:
                    pass
        res.append((d, units))
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    if traffic:
        d, units = res[0]

        def gb(k):
            v = float(d[k])
            return v * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12}.get(units[k], 1.0)

        tb = gb("dram__bytes_read.sum") + gb("dram__bytes_write.sum")
        info = {"kernel": d["Kernel Name"], "report": rep, "dram_bytes_per_launch": tb,
                "alg_bytes_per_launch": float(alg) if alg else None,
                "traffic_over_alg": tb / float(alg) if alg else None,
                "sm_ipc": float(d["sm__inst_executed.avg.per_cycle_active"]), "sm_ipc_peak": 4.0,
                "warp_instructions_per_launch": float(d["smsp__inst_executed.sum"]),
                "note": "top-level K3 launch of the C4 batch (tools/prof_batch.py 256), ncu --set full"}
        json.dump(info, open(traffic, "w"), indent=1)
        print(info)


def traffic(path, out, alg):
    """DRAM bytes of every K3 launch of one step (ncu --metrics dram__bytes_read.sum,
    dram__bytes_write.sum,gpu__time_duration.sum over the step's sweep launches)."""
    text = open(path).read()
    rd = csv.DictReader(io.StringIO(text[text.find('"ID"'):]))
    per = collections.defaultdict(dict)
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
             "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}
    for r in rd:
        per[r["ID"]][r["Metric Name"]] = float(r["Metric Value"].replace(",", "")) * scale.get(r["Metric Unit"], 1.0)
        per[r["ID"]]["name"] = r["Kernel Name"]
    launches_ = [v for _, v in sorted(per.items(), key=lambda x: int(x[0]))]
    tb = sum(v["dram__bytes_read.sum"] + v["dram__bytes_write.sum"] for v in launches_)
    info = {"kernel": launches_[0]["name"].split("(")[0], "launches_per_step": len(launches_),
            "dram_bytes_per_step": tb, "alg_bytes_per_step": float(alg), "traffic_over_alg": tb / float(alg),
            "per_launch": [{"dram_bytes": v["dram__bytes_read.sum"] + v["dram__bytes_write.sum"],
                            "ms_serialised": v.get("gpu__time_duration.sum")} for v in launches_],
            "source": path, "note": "every K3 launch of one C4 batch solve (tools/prof_batch.py 256), ncu "
                                    "--metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none"}
    json.dump(info, open(out, "w"), indent=1)
    print(json.dumps(info, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    elif sys.argv[1] == "traffic":
        traffic(*sys.argv[2:])
    else:
        full(*sys.argv[2:])
