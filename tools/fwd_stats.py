"""Diagnostic: per-warp time split of the forward kernel (TMA waits, unit prologue, unit
epilogue, compute) from a -DSKEI_FWD_STATS build (clock64 counters, printf from every 37th
CTA).  Builds the instrumented library under /tmp, runs one bench step through it.

    python tools/fwd_stats.py [--cta 37]
"""
import glob
import os
import re
import statistics as st
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2411_05771_b200")


def main():
    cta = int(sys.argv[sys.argv.index("--cta") + 1]) if "--cta" in sys.argv else 37
    lib = "/tmp/libskei_stats.so"
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                    "-Xcompiler", "-fPIC", "-shared", "--expt-relaxed-constexpr",
                    "-DSKEI_FWD_STATS", *os.environ.get("STATS_FLAGS", "").split(), "-I", os.path.join(ROOT, "include"), "-o", lib,
                    *sorted(glob.glob(os.path.join(PKG, "csrc", "*.cu")))], check=True)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "1",
                          "--warmup", "3", "--no-cpu-baseline", "--no-e2e"],
                         env=dict(os.environ, SKEI_LIB=lib), capture_output=True, text=True).stdout
    if os.environ.get("STATS_RAW"):  # keep the raw records (FWDSTAT per warp, FWDTASK per task)
        open(os.environ["STATS_RAW"], "w").write(out)
    rows = [list(map(int, re.findall(r"-?\d+", l))) for l in out.splitlines() if "FWDSTAT" in l]
    # cta warp units G wait pro epi total
    print("launch-CTA-warp records", len(rows), "median total cycles", st.median(r[7] for r in rows))
    for name, i in (("wait", 4), ("prologue", 5), ("epilogue", 6)):
        fr = [r[i] / r[7] for r in rows if r[7] > 0]
        print(f"{name:9s} median {st.median(fr):.3f} mean {st.mean(fr):.3f} max {max(fr):.3f}")
    last = [r for r in rows if r[0] == cta][-32:]
    seen = {}
    for r in last:
        seen[r[1]] = r
    for w in sorted(seen):
        r = seen[w]
        print(f"cta {r[0]} warp {w:2d} units {r[2]} blocks {r[3]} wait {r[4]:7d} pro {r[5]:6d} "
              f"epi {r[6]:6d} compute {r[7] - r[4] - r[5] - r[6]:7d} total {r[7]} "
              f"active tasks {r[8]} lanes/task {r[9] / max(1, r[8]):.1f}"
              + (f" esync {r[10]} fin {r[11]}" if len(r) > 11 else ""))


if __name__ == "__main__":
    main()
