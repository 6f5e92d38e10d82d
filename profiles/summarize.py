"""Rebuilds the launch-list / K1 tables of profiles/r1_summary.md and profiles/k1_traffic.json
from an ncu launch list (csv) and an `ncu --set full` capture of K1.
  python profiles/summarize.py <launches.csv> <k1.ncu-rep>"""
import collections
import csv
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))


def launch_table(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, rows = rows[0], rows[1:]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows:
        name = r[ki].split("(")[0].replace("void ", "").replace("gk::<unnamed>::", "").replace("<unnamed>::", "")[:70]
        tot[name] += float(r[vi].replace(",", ""))
        cnt[name] += 1
    total = sum(tot.values())
    lines = ["| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for n, t in sorted(tot.items(), key=lambda x: -x[1])[:16]:
        lines.append(f"| `{n}` | {cnt[n]} | {t / 1e6:.3f} | {100 * t / total:.1f}% |")
    return "\n".join(lines), len(rows)


def k1_tables(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(raw.splitlines()))
    h, u, v = r[0], r[1], r[2]
    m = {h[i]: (v[i], u[i]) for i in range(len(h))}
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
            "launch__registers_per_thread", "launch__grid_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__t_sector_hit_rate.pct",
            "lts__t_sector_hit_rate.pct", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
    k1 = ["| metric | value |", "|---|---|"] + [f"| `{k}` | {m[k][0]} {m[k][1]} |" for k in keys if k in m]
    st = sorted([(h[i], v[i]) for i in range(len(h)) if "warps_issue_stalled" in h[i] and h[i].endswith("per_issue_active.ratio")],
                key=lambda t: -float(t[1] or 0))[:7]
    stt = ["| stall | warps per issue |", "|---|---|"] + [
        f"| {n.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')} | {x} |" for n, x in st]
    scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}
    traffic = float(m["dram__bytes_read.sum"][0]) * scale[m["dram__bytes_read.sum"][1]] + \
        float(m["dram__bytes_write.sum"][0]) * scale[m["dram__bytes_write.sum"][1]]
    ms = float(m["gpu__time_duration.sum"][0]) * {"ms": 1, "us": 1e-3, "ns": 1e-6}[m["gpu__time_duration.sum"][1]]
    issue = float(m["smsp__issue_active.avg.pct_of_peak_sustained_active"][0])
    inst = float(m["smsp__inst_executed.sum"][0])
    return "\n".join(k1), "\n".join(stt), traffic, ms, issue, inst


if __name__ == "__main__":
    lt, n = launch_table(sys.argv[1])
    k1, st, traffic, ms, issue, inst = k1_tables(sys.argv[2])
    json.dump({"config": 2, "kernel": "k_knn<3,10>", "dram_bytes_per_launch": traffic,
               "issue_active_pct": issue, "warp_instructions": inst, "ncu_ms": ms,
               "source": "profiles/r1_summary.md (ncu --set full of the bench command)"},
              open(os.path.join(HERE, "k1_traffic.json"), "w"), indent=1)
    print(f"<!-- launches: {n} -->\n{lt}\n\n{k1}\n\n{st}\n\ntraffic {traffic / 1e9:.2f} GB, K1 {ms:.2f} ms")
