#!/bin/bash
# Round profile captures (run under gpurun, one GPU):
#   bench line, ncu launch list of the bench command, ncu --set full of the
#   numeric kernel of every config.  Output: gpurun_out/prof/
set -u
O=gpurun_out/prof
mkdir -p $O
python bench.py > $O/bench_default.log 2>&1; echo "bench rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench_cfg2.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_launches.log 2>&1; echo "launches rc=$?"
for c in 2 3 4 5; do
  case $c in 4) k=k_rows_ne3;; *) k=k_rows_tri;; esac
  ncu --set full --import-source on --clock-control none -k regex:$k -s 1 -c 1 -o $O/cfg${c}_$k \
      python tools/profile_step.py --config $c --reps 2 > $O/ncu_full_c$c.log 2>&1; echo "full c$c rc=$?"
done
for c in 2 3 4 5; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum \
      --clock-control none --csv --log-file $O/step_cfg$c.csv python tools/profile_step.py --config $c --reps 1 \
      > /dev/null 2>&1; echo "step c$c rc=$?"
done
