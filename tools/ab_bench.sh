#!/bin/bash
# A/B of two libskei builds through the same bench: tools/ab_bench.sh libA.so libB.so [reps]
A=$1; B=$2; N=${3:-3}
for r in $(seq $N); do
  for L in $A $B; do
    SKEI_LIB=$L timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$L'.split('/')[-1], round(d['value'],1), 'fwd', round(d['roofline']['kernel_ms']*1e3,1), 'us')"
  done
done
