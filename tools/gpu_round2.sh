#!/bin/bash
# Round-2 GPU session: GPU tests, default bench (config 5), per-pass DRAM traffic for the
# BASELINE configs, the bench's launch list, one full ncu capture of a config-5 forward
# chunk launch.  Usage: tools/gpu_round2.sh TAG [tests|bench|traffic|ncu]...
TAG=${1:-r02}; shift
STEPS=${*:-tests bench traffic ncu}
mkdir -p gpurun_out
for s in $STEPS; do case $s in
tests)
  NDC_PARITY_LOG=gpurun_out/parity_$TAG.jsonl timeout 1800 python -m pytest tests -m gpu -q -rfs --durations=15 \
      > gpurun_out/pytest_gpu_$TAG.log 2>&1
  echo "pytest rc=$?"; tail -25 gpurun_out/pytest_gpu_$TAG.log ;;
bench)
  timeout 1200 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
  echo "bench rc=$?"; cat gpurun_out/bench_$TAG.json; tail -3 gpurun_out/bench_$TAG.err ;;
traffic)
  for c in c5 c2 c3 c4; do
    timeout 600 python tools/ncu_traffic.py run $c > gpurun_out/counts_$c.json && \
    timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        --clock-control none --csv --log-file gpurun_out/traffic_${c}_$TAG.csv \
        python tools/ncu_traffic.py run $c > /dev/null 2> gpurun_out/traffic_${c}_$TAG.err
    echo "traffic $c rc=$?"
  done ;;
ncu)
  SHORT="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
  timeout 900 $SHORT > gpurun_out/short_$TAG.json 2>&1 && \
  # this repo's kernels only (namespace ndc::): the input generation (torch FFT / Poisson,
  # untimed setup) is not part of the measured step
  timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled \
      -k regex:"ndc::" -c 600 --csv --log-file gpurun_out/launches_$TAG.csv $SHORT > gpurun_out/ncu_launch_$TAG.log 2>&1
  echo "ncu launches rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:correlate -s 33 -c 1 \
      -o gpurun_out/prof_c5fwd_$TAG python tools/ncu_traffic.py run c5 > gpurun_out/ncu_full_$TAG.log 2>&1
  echo "ncu full rc=$?" ;;
esac; done
