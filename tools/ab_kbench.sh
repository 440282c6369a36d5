#!/bin/bash
# A/B kernel timing of library variants with SM clock / power sampled alongside.
# usage: tools/ab_kbench.sh "c2 c2k3" lib_old lib_new ...   (libs under tools/variants/;
# tools/variants/ is listed in .gpurunignore -- remove that line while running A/Bs on the GPU box)
CFGS=$1; shift
mkdir -p gpurun_out
nvidia-smi --query-gpu=timestamp,clocks.sm,power.draw,clocks_throttle_reasons.active --format=csv -lms 200 \
    > gpurun_out/ab_clocks.csv &
SMI=$!
for v in "$@"; do
  echo "== $v"
  NDC_LIB_PATH=tools/variants/$v.so python tools/kbench.py $CFGS
done
kill $SMI
