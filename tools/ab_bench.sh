#!/bin/bash
# A/B the libspx variants given as arguments with the default bench, interleaved
# (development; same box, same inputs).  Prints value, fused pass, final pass, convert.
#   bash tools/ab_bench.sh old new [rounds]
rounds=${3:-2}
for r in $(seq $rounds); do
  for v in "$1" "$2"; do
    SPX_LIB_VARIANT=variants/libspx_$v.so timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('$v', round(d['value']), 'fused %.4f final %.4f convert %.4f' % (r['mean_pass_ms'], r['final_assoc']['ms'], r['convert']['ms']), 'frac %.4f' % r['frac'])"
  done
done
