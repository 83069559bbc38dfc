#!/bin/bash
# A/B of prebuilt variants through bench.py --dist (P = 1 distributed step): tools/ab_dist.sh "A B" "5"
for c in ${2:-5}; do
  for n in ${1:-base A}; do
    cp vbuild/$n/libefem.so paper_1409_4618_b200/libefem.so
    timeout 300 python bench.py --dist --config $c --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('dist cfg$c $n', round(d['ms_per_step'],4))"
  done
done
