"""Build a variant of libskei.so with extra nvcc flags (A/B diagnostics):
    python tools/build_variant.py ab/libskei_x.so -DSKEI_FWD_KT4=5 ...
"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2411_05771_b200 import build as b  # noqa: E402

out, extra = sys.argv[1], sys.argv[2:]
cmd = [b.NVCC, *b.ARCH, *b.FLAGS, *extra, "-o", out, *b.sources()]
res = subprocess.run(cmd, capture_output=True, text=True)
if res.returncode:
    sys.exit(res.stdout + res.stderr)
for line in (res.stdout + res.stderr).splitlines():
    if "spill" in line and "radon_fwd" not in line:
        pass
print(out, "ok")
