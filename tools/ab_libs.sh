#!/bin/bash
# A/B the library builds in gpurun_out/ab on one command (development aid)
for v in base payload; do
  cp abtmp/$v.so paper_2402_13747_b200/libpcray_b200.so
  echo "== $v"; eval "$1"
done
