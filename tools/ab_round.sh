#!/bin/bash
# one A/B round under gpurun: ab_bench over the variants in $1 (configs $2),
# then the GPU tests with variant $3
bash tools/ab_bench.sh "$1" "$2" > gpurun_out/ab.txt 2>&1
cp vbuild/$3/libefem.so paper_1409_4618_b200/libefem.so
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/ab_tests.txt 2>&1; tail -2 gpurun_out/ab_tests.txt
cat gpurun_out/ab.txt
