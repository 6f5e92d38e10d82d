"""Digest of `ncu --set full` captures: one row per captured kernel launch with the
numbers DESIGN.md / the round summary cite (duration, DRAM bytes and GB/s, L2 read
sectors and hit rate, fp64 pipe, issue-active, warps active, instructions, registers,
shared memory, top stall reasons).

  python profiles/ncu_digest.py <report.ncu-rep> [...] [--md] [--k1-json profiles/k1_traffic.json --config N]

--k1-json writes the K1 (k_knn) launch's instruction count / DRAM bytes / issue share
with the hash of the K1 sources it was captured from; bench.py reads it for the
roofline's issue ceiling and marks it stale when the sources changed since."""
from __future__ import annotations

import csv
import hashlib
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
K1_SOURCES = ["paper_2207_01834_b200/csrc/gk_knn.cu", "paper_2207_01834_b200/csrc/gk_common.cuh"]


def k1_source_sha() -> str:
    h = hashlib.sha256()
    for f in K1_SOURCES:
        with open(os.path.join(ROOT, f), "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:16]


UNIT = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "Tbyte": 1e12,
        "ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1.0, "msecond": 1e-3, "usecond": 1e-6, "nsecond": 1e-9}


def rows_of(rep: str):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        if len(r) != len(h):
            continue
        d = {}
        for k, u, v in zip(h, units, r):
            try:
                x = float(v.replace(",", ""))
                d[k] = x * UNIT.get(u, 1.0)
            except ValueError:
                d[k] = v
        res.append(d)
    return res


STALLS = ["long_scoreboard", "wait", "short_scoreboard", "not_selected", "branch_resolving", "math_pipe_throttle",
          "lg_throttle", "mio_throttle", "barrier", "membar", "dispatch_stall", "no_instruction", "drain", "sleeping"]


def short_name(name: str) -> str:
    """'void gk::<unnamed>::k_knn<3, 10, 0>(gk::TreeSet, ...)' -> 'k_knn<3, 10, 0>'"""
    name = name.replace("void ", "").replace("<unnamed>", "anon").replace("unnamed>::", "")
    depth, cut = 0, len(name)
    for i, ch in enumerate(name):  # drop the argument list (the first '(' outside template brackets)
        depth += ch == "<"
        depth -= ch == ">"
        if ch == "(" and depth == 0:
            cut = i
            break
    name = name[:cut]
    base = name.split("<")[0]
    return base.split("::")[-1] + name[len(base):]


def digest(d: dict) -> dict:
    t = d.get("gpu__time_duration.sum", 0.0)
    rd, wr = d.get("dram__bytes_read.sum", 0.0), d.get("dram__bytes_write.sum", 0.0)
    st = {s: d.get(f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio", 0.0) for s in STALLS}
    top = sorted(st.items(), key=lambda kv: -kv[1])[:3]
    l2rd = d.get("lts__t_sectors_srcunit_tex_op_read.sum", 0.0) * 32
    name = str(d.get("Kernel Name", d.get("launch__kernel_name", "?")))
    return {
        "kernel": short_name(name),
        "ms": t * 1e3,
        "dram_read_gb": rd / 1e9, "dram_write_gb": wr / 1e9,
        "dram_gbs": (rd + wr) / t / 1e9 if t else None,
        "l2_read_gb": l2rd / 1e9, "l2_read_gbs": l2rd / t / 1e9 if t else None,
        "l2_hit_pct": d.get("lts__t_sector_hit_rate.pct"),
        "l1_hit_pct": d.get("l1tex__t_sector_hit_rate.pct"),
        "fp64_pipe_pct": d.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
        "issue_active_pct": d.get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "warps_active_pct": d.get("sm__warps_active.avg.pct_of_peak_sustained_active"),
        "warp_insts": d.get("smsp__inst_executed.sum"),
        "regs": d.get("launch__registers_per_thread"),
        "smem_kb": (d.get("launch__shared_mem_per_block_allocated") or 0) / 1e3 if isinstance(
            d.get("launch__shared_mem_per_block_allocated"), float) else d.get("launch__shared_mem_per_block_allocated"),
        "grid": d.get("launch__grid_size"), "block": d.get("launch__block_size"),
        "sm_ghz": d.get("sm__cycles_elapsed.avg.per_second", 0.0) / 1e9 if isinstance(
            d.get("sm__cycles_elapsed.avg.per_second"), float) else None,
        "top_stalls": [(k, round(v, 2)) for k, v in top],
    }


def md(rows):
    out = ["| kernel | ms | DRAM GB/s (frac of 6550) | DRAM R/W GB | L2 read GB/s | L2 hit % | L1 hit % | fp64 pipe % | "
           "issue % | warps % | regs | top stalls (warps/issue) |", "|" + "---|" * 12]
    for r in rows:
        f = lambda x, n=1: "-" if x is None else f"{x:.{n}f}"
        out.append(f"| `{r['kernel']}` | {f(r['ms'], 3)} | {f(r['dram_gbs'], 0)} ({f((r['dram_gbs'] or 0) / 6550.1, 2)}) | "
                   f"{f(r['dram_read_gb'], 3)} / {f(r['dram_write_gb'], 3)} | {f(r['l2_read_gbs'], 0)} | {f(r['l2_hit_pct'])} | "
                   f"{f(r['l1_hit_pct'])} | {f(r['fp64_pipe_pct'])} | {f(r['issue_active_pct'])} | {f(r['warps_active_pct'])} | "
                   f"{f(r['regs'], 0)} | " + ", ".join(f"{k} {v}" for k, v in r["top_stalls"]) + " |")
    return "\n".join(out)


def main(argv):
    reps = [a for a in argv if a.endswith(".ncu-rep")]
    rows = []
    for rep in reps:
        for d in rows_of(rep):
            r = digest(d)
            r["report"] = os.path.basename(rep)
            rows.append(r)
    if "--md" in argv:
        print(md(rows))
    else:
        for r in rows:
            print(json.dumps(r))
    if "--k1-json" in argv:
        path = argv[argv.index("--k1-json") + 1]
        cfg = int(argv[argv.index("--config") + 1]) if "--config" in argv else 2
        k1 = [r for r in rows if r["kernel"].startswith("k_knn")]
        if not k1:
            sys.exit("no k_knn launch in the capture")
        r = k1[0]
        json.dump({"config": cfg, "kernel": r["kernel"], "dram_bytes_per_launch": (r["dram_read_gb"] + r["dram_write_gb"]) * 1e9,
                   "l2_read_bytes_per_launch": r["l2_read_gb"] * 1e9,
                   "issue_active_pct": r["issue_active_pct"], "warp_instructions": r["warp_insts"], "ncu_ms": r["ms"],
                   "fp64_pipe_pct": r["fp64_pipe_pct"], "k1_source_sha": k1_source_sha(), "report": r["report"]},
                  open(path, "w"), indent=1)
        print("wrote", path)


if __name__ == "__main__":
    main(sys.argv[1:])
