#!/bin/bash
# the per-kernel step captures of tools/profile_round2.sh alone
set -u
O=gpurun_out/r2prof
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for c in 2 3 4 5; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum \
      --clock-control none --profile-from-start off --csv --log-file $O/step_cfg$c.csv \
      python tools/profile_step.py --config $c --reps 1 --warm 1 > /dev/null 2>&1; echo "step c$c rc=$?"
done
python tools/step_table.py $O/step_cfg2.csv $O/step_cfg3.csv $O/step_cfg4.csv $O/step_cfg5.csv > $O/step_tables.txt 2>&1
python tools/traffic_json.py $O > $O/traffic.json 2>&1
