#!/bin/bash
# A/B timing of prebuilt libefem.so variants under variants/<name>/:
#   tools/ab.sh "base A B" "4 2"   (configs)
names=${1:-"base A"}
cfgs=${2:-"4"}
mkdir -p gpurun_out
for c in $cfgs; do
  for n in $names; do
    cp vbuild/$n/libefem.so paper_1409_4618_b200/libefem.so
    timeout 300 python tools/time_numeric.py --config $c --tag $n 2>&1 | tail -1
  done
done
