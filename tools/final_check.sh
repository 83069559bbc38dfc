#!/bin/bash
# Full GPU validation of the current tree (run under gpurun, one GPU):
# build, pytest -m gpu, smoke(), then the round-2 evidence (tools/profile_round2.sh).
set -u
O=gpurun_out/final
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
timeout 1800 python -m pytest tests -m gpu -x -q --durations=15 > $O/gputests.log 2>&1; echo "pytest rc=$?"; tail -2 $O/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
bash tools/profile_round2.sh
