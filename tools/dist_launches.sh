#!/bin/bash
# per-kernel launch list of the P = 1 distributed step (bench.py --dist)
O=gpurun_out/dist; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $O/launches.csv python bench.py --dist --steps 2 --warmup 3 --no-cpu-baseline > $O/log 2>&1; echo rc=$?
