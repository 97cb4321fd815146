#!/bin/bash
# A/B device throughput of alternative engine builds in one GPU call.
# usage: scripts/ab.sh <preset> <count> lib1.so lib2.so ...
P=$1; N=$2; shift 2
for rep in 1 2; do
  for lib in "$@"; do
    echo "== $lib"
    HESP_LIB=$lib python scripts/probe_throughput.py $P $N 2>&1 | tail -1
  done
done
