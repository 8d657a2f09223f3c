#!/bin/bash
# A/B kernel timing on one box: scripts/ab_time.sh "<prof args>" lib1.so lib2.so ... (3 rounds, interleaved)
args=$1; shift
for r in 1 2 3; do
  for lib in "$@"; do
    printf "%-28s " "$(basename $lib)"; NACS_LIB=$(realpath $lib) python scripts/prof_batch.py $args 2>&1 | grep -o "requests: [0-9.]* ms"
  done
done
