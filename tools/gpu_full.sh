#!/bin/bash
# Full GPU test suite + bench per config (one gpurun call).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_full.log 2>&1
echo "full tests rc=$?"; tail -4 gpurun_out/gputests_full.log
bash tools/gpu_check.sh "${1:-2 3 4 5}" "abi_loads_nothing_matches_this" 2>&1 | grep -v "^tests\|deselected\|^$"
