#!/bin/bash
# Round-end measurement sweep: the headline line (with CPU baseline), the other configs, the
# next-row paths and the single-image splits on one GPU.  Output: gpurun_out/sweep/*.json
mkdir -p gpurun_out/sweep
python bench.py > gpurun_out/sweep/cfg3.json 2> gpurun_out/sweep/cfg3.err
for c in cfg2 cfg4 cfg5; do
  python bench.py --config $c --steps 30 --no-cpu-baseline > gpurun_out/sweep/$c.json 2> gpurun_out/sweep/$c.err
done
python bench.py --mode interleaved --no-cpu-baseline > gpurun_out/sweep/cfg3_il.json 2> gpurun_out/sweep/cfg3_il.err
for p in ei-grad rei deviation; do
  python bench.py --path $p --no-cpu-baseline > gpurun_out/sweep/$p.json 2> gpurun_out/sweep/$p.err
done
for s in angle angle-ag angle-p2p angle-rs; do
  python bench.py --config cfg5 --split $s --no-cpu-baseline --no-e2e > gpurun_out/sweep/cfg5_$s.json 2> gpurun_out/sweep/cfg5_$s.err
done
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/sweep/reference.json 2> gpurun_out/sweep/reference.err
