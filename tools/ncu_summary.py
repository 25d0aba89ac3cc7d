"""Summarise an ncu report (--set full) into the per-kernel numbers DESIGN.md and bench.py
cite: duration, DRAM/L2/shared-memory traffic, issue activity, occupancy, stall reasons.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep > profiles/<name>.txt
    python tools/ncu_summary.py gpurun_out/prof.ncu-rep --traffic profiles/ncu_traffic.json
"""
import csv
import io
import json
import re
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("lts__t_sectors.sum", "L2 sectors (32 B)"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "shared wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "shared bank conflicts"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/shared throughput %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("sm__cycles_elapsed.avg", "SM cycles"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__cluster_size", "cluster"),
    ("launch__occupancy_limit_registers", "occupancy limit (regs)"),
    ("launch__occupancy_limit_shared_mem", "occupancy limit (smem)"),
]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
        "msecond": 1e-3}


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def value(r, hdr, units, name):
    i = hdr.index(name)
    v = float(r[i].replace(",", ""))
    return v * UNIT.get(units[i], 1.0), units[i]


def main():
    rep = sys.argv[1]
    hdr, units, rows = load(rep)
    traffic = {}
    for r in rows:
        name = r[hdr.index("Kernel Name")]
        short = re.sub(r"\(.*", "", name).split("::")[-1]
        print(f"== {short}")
        for key, label in KEYS:
            if key not in hdr:
                continue
            v, u = value(r, hdr, units, key)
            if u in UNIT and UNIT[u] != 1.0 or u == "byte":
                unit = "s" if "second" in u else "B"
                print(f"   {label:28s} {v:16.6g} {unit}")
            else:
                print(f"   {label:28s} {v:16.6g} {u}")
        stalls = []
        for i, h in enumerate(hdr):
            m = re.match(r"smsp__average_warps_issue_stalled_(\w+)_per_issue_active\.ratio$", h)
            if m and r[i]:
                stalls.append((float(r[i].replace(",", "")), m.group(1)))
        stalls.sort(reverse=True)
        print("   stalls per issued instr    " + ", ".join(f"{n} {v:.2f}" for v, n in stalls[:6]))
        rd, _ = value(r, hdr, units, "dram__bytes_read.sum")
        wr, _ = value(r, hdr, units, "dram__bytes_write.sum")
        traffic.setdefault(short, rd + wr)
        for pre, stage in (("k_radon_fwd", "radon_fwd_x2"), ("k_radon_adj", "radon_adj_x2"),
                           ("k_ramp", "ramp"), ("k_rotate_pack", "rotate_pack")):
            if short.startswith(pre):
                traffic.setdefault(stage, rd + wr)
    if "--traffic" in sys.argv:
        path = sys.argv[sys.argv.index("--traffic") + 1]
        json.dump(traffic, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
