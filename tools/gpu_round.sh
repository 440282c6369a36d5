#!/bin/bash
# One GPU session: tests, bench, then (only after plain runs exit 0) ncu launch list +
# one full capture of the dominant kernel.  Usage: tools/gpu_round.sh [tag]
TAG=${1:-r01}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_$TAG.txt
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 600 > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench rc=$?"
cat gpurun_out/bench_$TAG.json
SHORT="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
if [ "${NCU:-1}" = "1" ]; then
  timeout 600 $SHORT > gpurun_out/short_$TAG.json 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv \
      --log-file gpurun_out/launches_$TAG.csv $SHORT > gpurun_out/ncu_launch_$TAG.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:correlate -s 10 -c 2 \
      -o gpurun_out/prof_$TAG $SHORT > gpurun_out/ncu_full_$TAG.log 2>&1
  echo "ncu rc=$?"
fi
