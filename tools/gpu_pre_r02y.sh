mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "vcycle or standalone or solve or warm or degenerate or gmres or full_size or fused" > gpurun_out/y_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/y_pytest.log
export MGM_TRACE=1
timeout 900 python tools/ab_solve.py - MGM_NO_MODE3=1 > gpurun_out/y_ab.jsonl 2> gpurun_out/y_ab.err
unset MGM_TRACE
timeout 300 python tools/standalone_time.py > gpurun_out/y_sa.jsonl 2>&1
