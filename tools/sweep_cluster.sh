for S in 0 1 2 3 4 6 8; do
  SKEI_FWD_CLUSTER=$S timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('S=$S', round(d['value'],1), 'fwd', round(d['roofline']['kernel_ms']*1e3,1), 'us')"
done
