#!/bin/bash
# A/B of several libskei builds through the same bench, interleaved: tools/ab_multi.sh reps lib...
N=$1; shift
for r in $(seq $N); do
  for L in "$@"; do
    SKEI_LIB=$L timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['stages_ms']; print('$L'.split('/')[-1], round(d['value'],1), 'fwd', round(d['roofline']['kernel_ms']*1e3,1), 'us', ' '.join(f'{k}={v*1e3:.1f}' for k,v in s.items()))"
  done
done
