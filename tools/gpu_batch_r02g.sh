mkdir -p gpurun_out
for rep in 1 2; do
for v in "MGM_X=0" "MGM_BATCH_CH8=1"; do
  echo "== $v" >> gpurun_out/b6_trace.txt
  env $v timeout 600 python tools/batch_trace.py 8 2>&1 | tail -1 >> gpurun_out/b6_trace.txt
  env $v timeout 600 python tools/batch_trace.py 4 2>&1 | tail -1 >> gpurun_out/b6_trace.txt
done
done
