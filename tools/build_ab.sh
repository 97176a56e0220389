#!/usr/bin/env bash
# Build experiment variants of the library for same-box A/B timing:
#   tools/build_ab.sh NAME="-DFLAG ..." [NAME2="..."]
# writes paper_2101_08763_b200/_ab/libNAME.so for each, then rebuilds the
# shipped library (no extra flags).  Load a variant with EXEM_LIB_PATH.
set -eu
cd "$(dirname "$0")/.."
mkdir -p paper_2101_08763_b200/_ab
for spec in "$@"; do
  name="${spec%%=*}"; flags="${spec#*=}"
  EXEM_NVCC_FLAGS="$flags" python -m paper_2101_08763_b200.build > /dev/null
  cp paper_2101_08763_b200/libexem_b200.so "paper_2101_08763_b200/_ab/lib$name.so"
  echo "built _ab/lib$name.so ($flags)"
done
python -m paper_2101_08763_b200.build > /dev/null
echo "shipped library rebuilt (flags: '$(cat paper_2101_08763_b200/libexem_b200.so.flags | tr -d '\n')')"
