#!/bin/bash
# A/B of library builds on C5 sequential scheduling: scripts/ab_c5.sh <method> <requests> lib1.so lib2.so ... (2 rounds, interleaved)
method=$1; nreq=$2; shift 2
for r in 1 2; do for lib in "$@"; do
  printf "%-14s " "$(basename $lib)"
  NACS_LIB=$(realpath $lib) timeout 120 python scripts/bench_c5.py --method $method --requests $nreq 2>&1 | tail -1 | cut -c1-400
done; done
