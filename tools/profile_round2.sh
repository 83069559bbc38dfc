#!/bin/bash
# Round-2 evidence (run under gpurun, one GPU): bench lines (default = config 5,
# every config, the reference arm), the ncu launch list of the default bench,
# per-kernel DRAM / time / instructions of one step per config, ncu --set full
# of the dominant kernels.  Output: gpurun_out/r2prof/
set -u
O=gpurun_out/r2prof
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
python bench.py --steps 20 --warmup 5 > $O/bench_default.log 2>&1; echo "bench rc=$?"
for c in 1 2 3 4 5; do
  python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline > $O/bench_c$c.log 2>&1; echo "bench c$c rc=$?"
done
python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_reference.log 2>&1; echo "ref rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench_default.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_launches.log 2>&1; echo "launches rc=$?"
for c in 2 3 4 5; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum \
      --clock-control none --profile-from-start off --csv --log-file $O/step_cfg$c.csv \
      python tools/profile_step.py --config $c --reps 1 --warm 1 \
      > /dev/null 2>&1; echo "step c$c rc=$?"
done
for spec in "5 k_rows_tri cfg5_k_rows_tri" "5 k_fan_nodes cfg5_k_fan_nodes" "2 k_rows_tri cfg2_k_rows_tri" \
            "4 k_rows_ne3 cfg4_k_rows_ne3" "3 k_rows_tri cfg3_k_rows_tri"; do
  set -- $spec
  ncu --set full --import-source on --clock-control none -k regex:$2 -s 1 -c 1 -o $O/$3 -f \
      python tools/profile_step.py --config $1 --reps 2 > $O/ncu_$3.log 2>&1; echo "full $3 rc=$?"
done
python tools/step_table.py $O/step_cfg2.csv $O/step_cfg3.csv $O/step_cfg4.csv $O/step_cfg5.csv > $O/step_tables.txt 2>&1
python tools/traffic_json.py $O > $O/traffic.json 2>&1
