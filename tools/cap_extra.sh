O=gpurun_out/cap
mkdir -p $O
for spec in "5 k_fan_fill_fixed cfg5_k_fan_fill" "4 k_node_count cfg4_k_node_count" "4 k_node_write cfg4_k_node_write"; do
  set -- $spec
  ncu --set full --import-source on --clock-control none -k regex:$2 -s 1 -c 1 -o $O/$3 -f \
      python tools/profile_step.py --config $1 --reps 2 > $O/ncu_$3.log 2>&1; echo "full $3 rc=$?"
done
