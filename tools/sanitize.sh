#!/bin/bash
# compute-sanitizer runs (memcheck, racecheck, synccheck, initcheck) over a representative
# subset of the GPU parity tests: every product kernel family launches at small sizes.
# Logs -> gpurun_out/sanitizer_<tool>.log; summary lines -> stdout.
SEL="test_gpu_gbt.py::test_predict_idx_bit_exact test_gpu_candidates.py::test_candidates_from_rows_matches_reference \
test_gpu_ppo.py test_gpu_sa.py::test_sa_spec_examples test_gpu_rollout.py::test_rollout_tc_edge_shapes \
test_gpu_rollout.py::test_rollout_bit_exact test_gpu_kmeans.py::test_kmeans_run_matches_reference \
test_gpu_kmeans.py::test_adaptive_sweep_and_snap_match_reference test_gpu_kmeans.py::test_snap_rule_fallback \
test_gpu_kmeans.py::test_assign_paths_bit_exact test_gpu_kmeans.py::test_certified_lloyd_rescue \
test_gpu_rollout.py::test_rollout_step_major_grouped test_gpu_rollout.py::test_rollout_tc_segmented_host_path \
test_gpu_rollout.py::test_rollout_ids_u32"
ARGS=""
for t in $SEL; do ARGS="$ARGS tests/$t"; done
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = "memcheck" ] && extra="--leak-check no"
  timeout 2400 compute-sanitizer --tool $tool $extra --target-processes all --error-exitcode 99 --print-limit 20 \
    python -m pytest $ARGS -x -q -p no:cacheprovider > gpurun_out/sanitizer_$tool.log 2>&1
  rc=$?
  echo "$tool rc=$rc: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|passed|failed' gpurun_out/sanitizer_$tool.log | tail -3 | tr '\n' ' ')"
done
