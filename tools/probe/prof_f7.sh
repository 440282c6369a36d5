#!/bin/bash
# ncu --set full of selected f7 probe launches (launch index = 4*config + 3)
cd "$(dirname "$0")"
for s in "$@"; do
  ncu --set full --clock-control none --import-source on -k k --launch-skip $s --launch-count 1 \
      -f -o ../../gpurun_out/f7prof_$s ./f7 > ../../gpurun_out/f7prof_$s.log 2>&1
  tail -1 ../../gpurun_out/f7prof_$s.log
done
