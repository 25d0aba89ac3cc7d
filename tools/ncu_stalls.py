"""Stall-reason breakdown of an ncu report's SASS source page, per reason and per hottest
instruction:  python tools/ncu_stalls.py rep.ncu-rep [kernel-regex] [--top N]"""
import csv, io, re, subprocess, sys
from collections import defaultdict


def main():
    rep = sys.argv[1]
    kre = sys.argv[2] if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else None
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 6
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    secs, cur = [], None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = [r[1] if len(r) > 1 else "", None, []]
            secs.append(cur)
        elif cur is not None and cur[1] is None:
            cur[1] = r
        elif cur is not None:
            cur[2].append(r)
    name, hdr, body = next(s for s in secs if kre is None or re.search(kre, s[0]))
    col = {h: i for i, h in enumerate(hdr)}
    reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = defaultdict(float)
    per = defaultdict(list)
    for r in body:
        for h in reasons:
            v = float(r[col[h]] or 0)
            if v:
                tot[h] += v
                per[h].append((v, r[col["Address"]], r[col["Source"]], r[col["Instructions Executed"]]))
    allv = sum(tot.values())
    print(name)
    for h, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"{h:28s} {v:8.0f} {100 * v / allv:5.1f}%")
        for v2, a, src, ex in sorted(per[h], reverse=True)[:top]:
            print(f"      {v2:6.0f}  {a}  x{ex:>9s}  {src.strip()[:70]}")


if __name__ == "__main__":
    main()
