#!/bin/bash
# In place of compute-sanitizer (closed on this pool): the canary tests and the
# parity / unstructured / edge-case GPU tests with EFEM_DEBUG_SYNC=1 (the library
# synchronises after every launch and reports the launch site of any error).
set -u
mkdir -p gpurun_out/guard
EFEM_DEBUG_SYNC=1 timeout 1500 python -m pytest tests -m gpu -q -x \
    -k "guards or parity_small or permuted or medium or unstructured or delaunay or fan or single or empty or range or bowtie or exact or dist2d" \
    > gpurun_out/guard/debug_sync_tests.log 2>&1
echo "debug-sync tests rc=$?"; tail -2 gpurun_out/guard/debug_sync_tests.log
