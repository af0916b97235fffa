mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "batch" > gpurun_out/b2_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/b2_pytest.log
timeout 600 python tools/batch_throughput.py > gpurun_out/b2_thr.json 2>&1
timeout 600 python tools/batch_trace.py 8 > gpurun_out/b2_trace8.txt 2>&1
MGM_BATCH_MORTON_T_MIN=1000000000000 timeout 600 python tools/batch_trace.py 8 > gpurun_out/b2_trace8_nomt.txt 2>&1
