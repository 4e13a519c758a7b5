#!/bin/bash
# A/B timing of alternative libsor builds on one box, interleaved (development aid):
#   tools/ab.sh "C3:4 C5:4 C3:4:solve" build/libsor_A.so build/libsor_B.so ...
specs="$1"; shift
for rep in 1 2; do
  for lib in "$@"; do
    SOR_LIBRARY=$lib timeout 300 python tools/ab_perf.py $specs
  done
done
