#!/bin/bash
# steady-state per-kernel step table of one config: tools/step_one.sh <config>
O=gpurun_out/stepone; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum \
    --clock-control none --profile-from-start off --csv --log-file $O/step_cfg$1.csv \
    python tools/profile_step.py --config $1 --reps 1 --warm 1 > /dev/null 2>&1; echo "rc=$?"
python tools/step_table.py $O/step_cfg$1.csv
