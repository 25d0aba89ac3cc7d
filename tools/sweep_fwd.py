"""Forward-projector timing sweep over cluster sizes (SKEI_FWD_CLUSTER), cfg3 shapes.
Prints one line per S: mean device time of skei_radon_fwd's forward launch (two jobs) via
the profiled pass.  Run on a GPU box: python tools/sweep_fwd.py"""
import json
import os
import subprocess
import sys

for S in range(1, 9):
    env = dict(os.environ, SKEI_FWD_CLUSTER=str(S))
    out = subprocess.run([sys.executable, "bench.py", "--steps", "30", "--warmup", "5",
                          "--no-cpu-baseline", "--no-e2e"], env=env, capture_output=True, text=True)
    try:
        d = json.loads(out.stdout.strip().splitlines()[-1])
        print(f"S={S} fwd_ms={d['stages_ms']['radon_fwd_x2']:.4f} passes/s={d['value']:.1f}", flush=True)
    except Exception:
        print(f"S={S} failed: {out.stderr[-300:]}", flush=True)
