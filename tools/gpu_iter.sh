#!/bin/bash
# quick iteration: build, GPU tests (optionally filtered), bench lines for the given configs
#   tools/gpu_iter.sh "<pytest -k expr or empty>" "5 2" [steps]
set -u
O=gpurun_out/iter
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo "build failed"; tail -20 $O/build.log; exit 1; }
K="${1:-}"
if [ -n "$K" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q -k "$K" > $O/tests.log 2>&1; echo "tests rc=$?"; tail -3 $O/tests.log
elif [ "$K" != "none" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > $O/tests.log 2>&1; echo "tests rc=$?"; tail -3 $O/tests.log
fi
for c in ${2:-5}; do
  timeout 600 python bench.py --config $c --steps ${3:-50} --warmup 5 --no-cpu-baseline > $O/bench_c$c.log 2>&1
  echo "bench c$c rc=$?"; tail -1 $O/bench_c$c.log | cut -c1-400
done
