#!/bin/bash
# fused one-call kernel vs the separate fan pass + row kernel (EFEM_FUSED=0)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in ${1:-5 2}; do
  for f in 0 1; do
    EFEM_FUSED=$f timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('cfg$c fused=$f', round(d['ms_per_step'],4), round(d['roofline']['frac'],3))"
  done
done
