#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over tools/sanitize_case.py
# (through gpurun); logs -> gpurun_out/sanitize/<tool>_<case>.log, summary on stdout.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/sanitize
CS=compute-sanitizer
for tool in memcheck synccheck racecheck initcheck; do
  for c in c1a tiny3d_cl_fluid c3; do
    extra=""
    [ "$tool" = memcheck ] && extra="--leak-check full"
    [ "$tool" = racecheck ] && extra="--racecheck-report all"
    steps=6; [ "$tool" = racecheck ] && steps=2
    SAN_STEPS=$steps timeout 900 $CS --tool $tool $extra --error-exitcode 9 python tools/sanitize_case.py $c \
      > gpurun_out/sanitize/${tool}_${c}.log 2>&1
    echo "$tool $c exit=$? :: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|LEAK SUMMARY' gpurun_out/sanitize/${tool}_${c}.log | tr '\n' ' ')"
  done
done
