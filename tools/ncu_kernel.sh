#!/bin/bash
# ncu --set full of one kernel of one assembly step: tools/ncu_kernel.sh <config> <kernel regex> <name>
set -u
mkdir -p gpurun_out/ncu
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:$2 -s 1 -c 1 -o gpurun_out/ncu/$3 -f \
    python tools/profile_step.py --config $1 --reps 2 > gpurun_out/ncu/$3.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/ncu/$3.ncu-rep --page details --csv > gpurun_out/ncu/$3_details.csv 2>&1
