#!/bin/bash
# Round-2 measurement call: GPU suite, the sweep, the launch list and one full capture of the
# pass kernels.  Usage (on the box): bash tools/r2_measure.sh TAG [skip-tests]
TAG=${1:-r2}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_throttle_reasons.active --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || { echo BUILD FAILED; tail gpurun_out/${TAG}_build.log; exit 1; }
if [ "$2" != "skip-tests" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_gputests.log 2>&1
  echo "gpu tests rc=$?"; tail -3 gpurun_out/${TAG}_gputests.log
  timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
  echo "smoke rc=$?"; tail -1 gpurun_out/${TAG}_smoke.log
fi
bash tools/sweep.sh
mkdir -p gpurun_out/${TAG}_sweep && mv gpurun_out/sweep/* gpurun_out/${TAG}_sweep/
for f in gpurun_out/${TAG}_sweep/*.json; do echo "$f: $(head -c 400 $f)"; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e \
  > gpurun_out/${TAG}_ncu_launch.log 2>&1
echo "ncu launch rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ -s 30 -c 10 \
  -o gpurun_out/${TAG}_full -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e \
  > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "ncu full rc=$?"
