# compute-sanitizer memcheck (one tool per call) over the round-2 code paths on small clouds
mkdir -p gpurun_out
timeout 2400 compute-sanitizer --tool memcheck --error-exitcode 17 --print-limit 20 \
  python -m pytest tests/test_gpu_parity.py -m gpu -q -x \
  -k "dist_fake_ranks_vcycle_bitwise or (dist_fake_ranks_solve and torus20000 and 1) or (dense_bottom and cfg1) or (warm_start_x0 and cfg1) or (structures_exact and poisson6000) or spgemm_long or (vcycle and cfg1) or zero_rhs or degenerate" \
  > gpurun_out/sanitize.log 2>&1
echo "sanitize rc=$?" >> gpurun_out/sanitize.log
