"""Per-opcode / hottest-instruction view of an ncu report's SASS source page.

    python tools/ncu_sass.py gpurun_out/prof.ncu-rep [kernel-regex] [--top N]
"""
import csv
import io
import re
import subprocess
import sys
from collections import Counter


def main():
    rep = sys.argv[1]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 30
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    kre = sys.argv[2] if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else None
    # the page holds one section per kernel: ["Kernel Name", name], header, rows...
    secs, cur = [], None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = [r[1] if len(r) > 1 else "", None, []]
            secs.append(cur)
        elif cur is not None and cur[1] is None:
            cur[1] = r
        elif cur is not None:
            cur[2].append(r)
    sec = next(s for s in secs if kre is None or re.search(kre, s[0]))
    print("kernel:", sec[0][:100])
    hdr, rows = sec[1], [None, None] + sec[2]
    isrc, iex = hdr.index("Source"), hdr.index("Instructions Executed")
    iss = hdr.index("Warp Stall Sampling (All Samples)")
    iwf = hdr.index("L1 Wavefronts Shared") if "L1 Wavefronts Shared" in hdr else None
    c, s, w = Counter(), Counter(), Counter()
    hot = []
    for r in rows[2:]:
        if len(r) <= iex or not r[iex]:
            continue
        src = r[isrc].strip()
        op = re.sub(r"^@!?U?P\w+\s+", "", src).split()[0] if src else "?"
        ex, st = int(r[iex] or 0), int(r[iss] or 0)
        c[op] += ex
        s[op] += st
        if iwf is not None and r[iwf]:
            w[op] += int(float(r[iwf]))
        hot.append((st, ex, src))
    tot, tst = sum(c.values()), max(1, sum(s.values()))
    print(f"total warp instructions {tot}, stall samples {tst}")
    for op, v in c.most_common(top):
        print(f"  {op:24s} {v:>11d} {100 * v / tot:5.1f}%  stall {100 * s[op] / tst:5.1f}%  smem_wf {w[op]}")
    print("hottest instructions by stall samples:")
    for st, ex, src in sorted(hot, reverse=True)[:top]:
        print(f"  {st:>6d} {ex:>10d}  {src[:100]}")


if __name__ == "__main__":
    main()
