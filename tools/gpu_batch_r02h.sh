mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "batch" > gpurun_out/b7_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/b7_pytest.log
timeout 600 python tools/batch_throughput.py > gpurun_out/b7_thr.json 2>&1
for K in 2 4 8; do timeout 600 python tools/batch_trace.py $K 2>&1 | tail -1 >> gpurun_out/b7_trace.txt; done
MGM_BATCH_CH8=1 timeout 600 python tools/batch_trace.py 2 2>&1 | tail -1 >> gpurun_out/b7_trace.txt
