"""Per-launch table (time, DRAM bytes and GB/s, fp64 pipe and issue utilisation) from an
`ncu --set full` capture:  python profiles/kernel_table.py <report.ncu-rep>"""
import csv
import subprocess
import sys

COLS = [("gpu__time_duration.sum", "ms", 1e-6), ("dram__bytes_read.sum", "rd MB", 1e-6),
        ("dram__bytes_write.sum", "wr MB", 1e-6), ("launch__grid_size", "grid", 1),
        ("launch__registers_per_thread", "regs", 1),
        ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe %", 1),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %", 1),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps %", 1)]
UNIT = {"ns": 1, "us": 1e3, "ms": 1e6, "nsecond": 1, "usecond": 1e3, "msecond": 1e6, "s": 1e9,
        "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, u = rows[0], rows[1]
    print("| kernel | " + " | ".join(c[1] for c in COLS) + " | DRAM GB/s |")
    print("|---" * (len(COLS) + 2) + "|")
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "").replace("gk::<unnamed>::", "")
        vals, raw_v = [], {}
        for key, _, scale in COLS:
            i = h.index(key)
            v = float(r[i].replace(",", "")) * UNIT.get(u[i], 1)
            raw_v[key] = v
            vals.append(f"{v * scale:.3f}" if scale != 1 else f"{v:.1f}")
        t = raw_v["gpu__time_duration.sum"]
        gbs = (raw_v["dram__bytes_read.sum"] + raw_v["dram__bytes_write.sum"]) / t if t else 0.0
        print(f"| `{name[:40]}` | " + " | ".join(vals) + f" | {gbs:.0f} |")


if __name__ == "__main__":
    main(sys.argv[1])
