mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "batch or dense" > gpurun_out/j_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/j_pytest.log
for v in "MGM_X=0" "MGM_DENSE_SPLIT=1" "MGM_DENSE_SPLIT=8"; do
  echo "== $v" >> gpurun_out/j_trace.txt
  for K in 4 8; do env $v timeout 600 python tools/batch_trace.py $K 2>&1 | tail -1 >> gpurun_out/j_trace.txt; done
done
timeout 600 python tools/batch_throughput.py > gpurun_out/j_thr.json 2>&1
