"""Summarise an ncu CSV (--csv --page raw style metrics, one row per launch) of
tools/profile_step.py into profiles/far_kernel_ncu.json: DRAM bytes, time and
FP64-pipe activity of the far-field launches (k_m2p_far + k_cheb_*) of the
LAST fast product in the capture.

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,\
sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread \
        --clock-control none --csv --log-file far.csv python tools/profile_step.py
    python tools/far_ncu_summary.py far.csv profiles/far_kernel_ncu.json
"""
import csv
import json
import re
import sys
from collections import OrderedDict


def main(src, dst):
    rows = [r for r in csv.reader(open(src)) if len(r) > 10]
    hdr = rows[0]
    col = {k: hdr.index(k) for k in ("ID", "Kernel Name", "Grid Size", "Metric Name", "Metric Unit",
                                     "Metric Value")}
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}
    launches = OrderedDict()
    for r in rows[1:]:
        d = launches.setdefault(r[col["ID"]], {"name": r[col["Kernel Name"]],
                                               "grid": r[col["Grid Size"]]})
        v = float(r[col["Metric Value"]].replace(",", ""))
        if r[col["Metric Name"]] == "gpu__time_duration.sum":
            v *= scale.get(r[col["Metric Unit"]], 1e-6) * 1e6  # -> ns
        d[r[col["Metric Name"]]] = v
    seq = list(launches.values())
    starts = [i for i, d in enumerate(seq) if re.search(r"k_gather\b", d["name"]) and "rows" not in d["name"]]
    last = seq[starts[-1]:] if starts else seq
    far = [d for d in last if re.search(r"k_m2p_far|k_m2p_leaf2|k_node_gemm", d["name"])]
    cheb = [d for d in last if "k_cheb" in d["name"]]
    ms = lambda d: d.get("gpu__time_duration.sum", 0.0) / 1e6
    dram = lambda d: d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    out = {
        "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,"
                  "sm__pipe_fp64_cycles_active... --clock-control none, tools/profile_step.py (cfg4), "
                  "last of 3 products; summarised by tools/far_ncu_summary.py",
        "kernel": "k_m2p_far / k_m2p_leaf2 / k_node_gemm (node, ring, X-node and partial passes of "
                  "one fast product) and the k_cheb_* kernels",
        "dram_bytes_per_launch": sum(dram(d) for d in far),
        "ncu_ms": sum(ms(d) for d in far),
        "launches": len(far),
        "with_cheb_kernels": {"dram_bytes": sum(dram(d) for d in far + cheb),
                              "ms": sum(ms(d) for d in far + cheb)},
        "per_launch": [{"name": re.sub(r"\(.*", "", d["name"]), "grid": d["grid"], "ms": ms(d),
                        "fp64_pipe_pct": d.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
                        "tensor_pipe_pct": d.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
                        "dram_read": d.get("dram__bytes_read.sum"),
                        "dram_write": d.get("dram__bytes_write.sum"),
                        "regs": d.get("launch__registers_per_thread")} for d in far + cheb],
    }
    json.dump(out, open(dst, "w"), indent=1)
    print(f"{len(far)} far launches, {out['ncu_ms']:.2f} ms, {out['dram_bytes_per_launch'] / 1e9:.2f} GB")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
