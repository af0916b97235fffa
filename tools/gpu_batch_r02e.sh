# RHS-split batched kernels: parity, then K = 4 / 8 traced and throughput A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "batch" > gpurun_out/b_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/b_pytest.log
for v in 1 0; do
  MGM_BATCH_SPLIT=$v timeout 600 python tools/batch_throughput.py > gpurun_out/b_thr_$v.json 2>&1
  MGM_BATCH_SPLIT=$v timeout 600 python tools/batch_trace.py 8 > gpurun_out/b_trace8_$v.txt 2>&1
done
