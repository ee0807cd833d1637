#!/bin/bash
# A/B the kernel variants in variants/ with the default bench (development).
for lib in variants/libspx_*.so; do
  SPX_LIB_VARIANT=$lib timeout 300 python bench.py --steps 10 --warmup 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']['stage_ms']; print('$lib', round(d['value']), [round(x,3) for x in r['associate']], round(r['update'][0],3))"
done
