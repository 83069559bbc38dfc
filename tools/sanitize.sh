#!/bin/bash
# compute-sanitizer (memcheck, racecheck, initcheck, synccheck) over small
# end-to-end assemblies (tools/tiny.py: symbolic + numeric + check) of every
# element kind, config 1, a config-2-shaped 2D mesh, and scipy Delaunay
# meshes; SURVEY.md §5.  Logs: gpurun_out/sanitize/<tool>_<case>.log
set -u
O=gpurun_out/sanitize
mkdir -p $O
CASES="2,0,16 2,1,48 2,0,130 3,0,5 3,1,5 3,0,9 3,1,9 dl2,0,0 dl2,1,0 dl3,0,0 dl3,1,0"
for tool in memcheck racecheck initcheck synccheck; do
  for c in $CASES; do
    IFS=, read d e n <<< "$c"
    timeout 900 compute-sanitizer --tool $tool --error-exitcode 99 --print-limit 20 \
        python tools/tiny.py $d $e $n > $O/${tool}_${d}_${e}_${n}.log 2>&1
    echo "$tool $d $e $n rc=$? $(grep -h 'ERROR SUMMARY' $O/${tool}_${d}_${e}_${n}.log | tail -1)"
  done
done
