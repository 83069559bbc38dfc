#!/bin/bash
# Per-kernel time / DRAM bytes of one assembly step for the given configs:
#   tools/step_profile.sh "3 4"  -> gpurun_out/step_cfg<c>.csv
mkdir -p gpurun_out
for c in ${1:-4}; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum \
      --clock-control none --csv --log-file gpurun_out/step_cfg$c.csv python tools/profile_step.py --config $c --reps 1 \
      > /dev/null 2>&1; echo "step c$c rc=$?"
done
