#!/bin/bash
# A/B of libskei builds over several configs: tools/ab_cfgs.sh "cfg3 cfg4 cfg5" lib...
CFGS=$1; shift
for c in $CFGS; do
  for L in "$@"; do
    SKEI_LIB=$L timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-e2e | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['stages_ms']; print('$c', '$L'.split('/')[-1], round(d['value'],1), ' '.join(f'{k}={v*1e3:.1f}' for k,v in s.items()))"
  done
done
