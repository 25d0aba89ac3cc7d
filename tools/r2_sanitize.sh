#!/bin/bash
# One compute-sanitizer tool per gpurun call (B200_PROFILING.md): bash tools/r2_sanitize.sh TOOL [args]
TOOL=$1; shift
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/san_build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 300 python tools/sanitize_run.py "$@" > gpurun_out/san_plain_${TOOL}.log 2>&1
rc=$?; echo "plain rc=$rc"; tail -2 gpurun_out/san_plain_${TOOL}.log
[ $rc -eq 0 ] || exit 1
timeout 1500 compute-sanitizer --tool $TOOL --print-limit 50 python tools/sanitize_run.py "$@" > gpurun_out/san_${TOOL}.log 2>&1
echo "sanitizer rc=$?"; tail -8 gpurun_out/san_${TOOL}.log
