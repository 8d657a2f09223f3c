#!/bin/bash
# Build libnacs.so of git revision $1 into exp/$2.so (A/B timing on one box with NACS_LIB).
set -e
rev=$1; name=$2
root=$(cd "$(dirname "$0")/.." && pwd)
tmp=$(mktemp -d)
git -C "$root" archive "$rev" paper_1909_07673_b200 include | tar -x -C "$tmp"
mkdir -p "$root/exp"
(cd "$tmp" && python paper_1909_07673_b200/build.py "$root/exp/$name.so")
rm -rf "$tmp"
echo "built exp/$name.so from $rev"
