#!/bin/bash
# A/B of library builds on one gpurun call (development aid): copy each variant to
# abtmp/<name>.so (git-ignored, travels with the snapshot), then
#   tools/ab_libs.sh "<command>" name1 name2 ...
cmd="$1"; shift
for v in "$@"; do
  cp "abtmp/$v.so" paper_2402_13747_b200/libpcray_b200.so
  echo "== $v"; eval "$cmd"
done
