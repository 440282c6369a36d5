#!/bin/bash
# compute-sanitizer over the KAT-sized GPU cases that exercise the risky machinery:
# chunked tap accumulation through scratch, edge-tile launches on the side stream
# (compact lane mapping, tap-row phases folded through shared memory), packed FFMA2
# widths, the speculative next-step adjoint with staggered stops, the in-process z-slab
# ranks (halo exchange on the comm stream) and the one-rank NCCL transport.
# Usage: tools/sanitize.sh memcheck|racecheck|synccheck|initcheck [TAG]
TOOL=$1; TAG=${2:-r02}
mkdir -p gpurun_out
CASES="tests/test_gpu_ops.py::test_large_psfs_chunked tests/test_gpu_ops.py::test_edge_tiles_few_rows
 tests/test_gpu_ops.py::test_packed_ffma2_widths tests/test_gpu_pg.py::test_batch_staggered_stops_vs_oracle
 tests/test_gpu_pg.py::test_acceptance6_backtracking tests/test_gpu_sharded.py::test_sharded_pg_matches_unsharded
 tests/test_gpu_nccl.py::test_nccl_single_rank_matches_unsharded"
EXTRA=""
[ "$TOOL" = "memcheck" ] && EXTRA="--leak-check full"
timeout 3000 /usr/local/cuda/bin/compute-sanitizer --tool $TOOL $EXTRA --target-processes all \
    --error-exitcode 99 --log-file gpurun_out/sanitize_${TOOL}_$TAG.%p.log \
    python -m pytest $CASES -q -p no:cacheprovider > gpurun_out/sanitize_${TOOL}_$TAG.pytest.log 2>&1
echo "sanitizer $TOOL rc=$?"
tail -3 gpurun_out/sanitize_${TOOL}_$TAG.pytest.log
for f in gpurun_out/sanitize_${TOOL}_$TAG.*.log; do echo "== $f"; grep -E "ERROR SUMMARY|LEAK SUMMARY|Hazard|Error" $f | sort | uniq -c | head -20; done
