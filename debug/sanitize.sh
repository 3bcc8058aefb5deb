#!/bin/bash
# compute-sanitizer (memcheck / racecheck / synccheck / initcheck) over the
# small-shape GPU tests that reach every kernel of the library.
#   bash debug/sanitize.sh [tool ...]   -> gpurun_out/sanitize_<tool>.log
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TESTS="tests/test_gpu_forward.py::test_ragged_shapes tests/test_gpu_forward.py::test_mini_arch_simt
tests/test_gpu_forward.py::test_pbm_payload_matches_packbits tests/test_gpu_forward.py::test_fused_pass_plans_for_other_depths
tests/test_gpu_forward.py::test_row_window_sharding_bitwise tests/test_gpu_forward.py::test_nonfinite_logits_raise
tests/test_gpu_conv_tc.py tests/test_gpu_wgrad_tc.py::test_wgrad_vs_fp64
tests/test_gpu_train.py::test_forward_backward_vs_reference tests/test_gpu_train.py::test_reward_delta_le
tests/test_gpu_train.py::test_anisotropy_loss_and_grad tests/test_gpu_train.py::test_rapsd_of_halftone
tests/test_gpu_train.py::test_adam_matches_reference tests/test_gpu_train.py::test_make_sample_draw_order_and_le
tests/test_rng.py::test_device_uniforms_bit_exact tests/test_rng.py::test_device_gaussians_match_host_stream
tests/test_rng.py::test_gaussian_maps_from_recorded_states
tests/test_estimators.py::test_device_binary_signals tests/test_estimators.py::test_device_reinforce_signals
tests/test_estimators.py::test_device_multitone_sample_and_le tests/test_estimators.py::test_multitone_inference_matches_oracle"
tools=${@:-memcheck racecheck synccheck initcheck}
for t in $tools; do
  extra=""
  [ "$t" = "memcheck" ] && extra="--leak-check no"
  timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $t $extra --kernel-name-exclude regex:at:: \
    --print-limit 20 python -m pytest -q -x -m gpu -p no:cacheprovider $TESTS > gpurun_out/sanitize_$t.log 2>&1
  echo "$t rc=$? $(grep -E 'ERROR SUMMARY|passed|failed' gpurun_out/sanitize_$t.log | tr '\n' ' ')"
done
