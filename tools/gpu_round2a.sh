set -u
mkdir -p gpurun_out/r2a
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2a/build.log 2>&1
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/fp64_peak tools/fp64_peak.cu && /tmp/fp64_peak > gpurun_out/r2a/fp64_peak.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q --durations=25 > gpurun_out/r2a/gputests.log 2>&1; echo "pytest rc=$?"
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/r2a/bench_default.log 2>&1; echo "bench rc=$?"
timeout 1200 bash tools/sanitize.sh > gpurun_out/r2a/sanitize_summary.txt 2>&1; echo "san rc=$?"
cp -r gpurun_out/sanitize gpurun_out/r2a/ 2>/dev/null
