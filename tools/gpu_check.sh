#!/bin/bash
# One gpurun round trip: GPU tests, then the bench on the given configs.
#   tools/gpu_check.sh "2 3 5" [pytest -k expr]
cfgs=${1:-"2"}
kexpr=${2:-}
mkdir -p gpurun_out
if [ -n "$kexpr" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q -k "$kexpr" > gpurun_out/gputests.log 2>&1
else
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1
fi
echo "tests rc=$?"; tail -15 gpurun_out/gputests.log | grep -v "^$"
for c in $cfgs; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c$c.log 2>&1
  echo "c$c rc=$?"
  python - "$c" <<'PY'
import json,sys
c=sys.argv[1]
try:
    line=[l for l in open(f"gpurun_out/bench_c{c}.log") if l.startswith("{")][-1]
    d=json.loads(line)
    print(f"cfg{c}: {d['ms_per_step']:.4f} ms/step  {d['value']/1e9:.3f} Gelem/s  phases {d['phase_ms']}  numeric frac {d['roofline']['frac']:.3f}  e2e_frac {d['roofline']['e2e_frac']:.3f}")
except Exception as ex:
    print("no result", ex); print(open(f"gpurun_out/bench_c{c}.log").read()[-2000:])
PY
done
