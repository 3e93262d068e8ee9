"""Per-launch table of an `ncu --set full` capture exported with
`ncu -i X.ncu-rep --page raw --csv` (one row per launch, one column per
metric): time, FP64 / tensor pipe activity, issue slots, DRAM bytes,
registers, occupancy and the top warp-stall reasons.

    python tools/ncu_full_summary.py raw.csv > profiles/rNN_ncu_full_summary.md
"""
import csv
import re
import sys

COLS = [
    ("ms", "gpu__time_duration.sum", 1e-6),
    ("fp64 pipe %", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 1),
    ("fp64 inst %", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", 1),
    ("tensor pipe %", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 1),
    ("issue %", "smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    ("warps %", "sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    ("regs", "launch__registers_per_thread", 1),
    ("DRAM rd MB", "dram__bytes_read.sum", 1e-6),
    ("DRAM wr MB", "dram__bytes_write.sum", 1e-6),
    ("DRAM %", "dram__throughput.avg.pct_of_peak_sustained_elapsed", 1),
]


def num(s):
    try:
        return float(s.replace(",", ""))
    except ValueError:
        return None


def main(src):
    rows = list(csv.reader(open(src)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hd, units = rows[h], rows[h + 1]
    data = [r for r in rows[h + 2:] if len(r) == len(hd)]
    ix = {k: i for i, k in enumerate(hd)}
    stall = [k for k in hd if re.match(r"smsp__average_warps_issue_stalled_.*_per_issue_active\.ratio$", k)
             or re.match(r"smsp__average_warp_latency_issue_stalled_.*\.ratio$", k)]
    if not stall:
        stall = [k for k in hd if "issue_stalled" in k and k.endswith(".ratio")]
    tscale = {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}
    print("| # | kernel | grid | " + " | ".join(c[0] for c in COLS) + " | top stalls (warps per issue) |")
    print("|" + "---|" * (len(COLS) + 4))
    tot = 0.0
    for n, r in enumerate(data):
        name = re.sub(r"\(.*", "", r[ix["Kernel Name"]])
        name = re.sub(r"^void |imqk::|<?unnamed>::|\(anonymous namespace\)::", "", name)
        cells = []
        for label, key, sc in COLS:
            if key not in ix:
                cells.append("-")
                continue
            v = num(r[ix[key]])
            if v is None:
                cells.append("-")
                continue
            if label == "ms":
                v *= tscale.get(units[ix[key]], 1e-6)
                tot += v
                cells.append(f"{v:.3f}")
            elif label.startswith("DRAM") and "MB" in label:
                u = units[ix[key]].lower()
                mul = {"byte": 1e-6, "kbyte": 1e-3, "mbyte": 1.0, "gbyte": 1e3}.get(u, 1e-6)
                cells.append(f"{v * mul:.1f}")
            else:
                cells.append(f"{v:.1f}" if label != "regs" else f"{int(v)}")
        st = []
        for k in stall:
            v = num(r[ix[k]])
            if v:
                st.append((v, re.sub(r".*issue_stalled_(.*?)(_per_issue_active)?\.ratio", r"\1", k)))
        st.sort(reverse=True)
        top = ", ".join(f"{nm} {v:.2f}" for v, nm in st[:3])
        grid = r[ix["Grid Size"]] if "Grid Size" in ix else ""
        print(f"| {n} | `{name}` | {grid} | " + " | ".join(cells) + f" | {top} |")
    print(f"\ntotal {tot:.3f} ms over {len(data)} launches (serialised, under ncu replay)")


if __name__ == "__main__":
    main(sys.argv[1])
