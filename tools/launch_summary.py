"""Per-kernel launch list summary of an `ncu --metrics gpu__time_duration.sum --csv` log:
launches, mean device time, and each pass kernel's share of the per-step sum.

    python tools/launch_summary.py gpurun_out/launches.csv "header line" > profiles/<name>.txt
"""
import csv
import re
import sys
from collections import OrderedDict

PASS = ["k_draw", "k_rotate_pack", "k_radon_fwd", "k_ramp", "k_radon_adj"]


def main():
    rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
    hdr = rows[0]
    ci = {h: i for i, h in enumerate(hdr)}
    per = OrderedDict()
    for r in rows[1:]:
        if r[ci["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*$", "", r[ci["Kernel Name"]])
        name = re.sub(r"^void |skei::|<unnamed>::|\(anonymous namespace\)::|at::", "", name).strip()
        v = float(r[ci["Metric Value"]].replace(",", ""))
        unit = r[ci["Metric Unit"]]
        v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3,
              "msecond": 1e3}.get(unit, 1.0)
        per.setdefault(name, []).append(v)
    for line in sys.argv[2:]:
        print("# " + line)
    print("# per-launch device time, cold-cache and serialised: compare shares, not absolutes")
    for k, v in per.items():
        print(f"{k:40s} launches={len(v):3d} mean_us={sum(v) / len(v):9.1f}")
    pk = [k for k in per if any(k.startswith(p) for p in PASS)]
    tot = sum(sum(per[k]) / len(per[k]) for k in pk)
    print(f"# pass total (sum of the {len(pk)} per-step kernel means) = {tot:.1f} us")
    for k in pk:
        print(f"#   share {k:28s} {100 * sum(per[k]) / len(per[k]) / tot:5.1f} %")


if __name__ == "__main__":
    main()
