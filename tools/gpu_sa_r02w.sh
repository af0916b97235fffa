mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "standalone or solve or warm or degenerate or gmres" > gpurun_out/w_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/w_pytest.log
timeout 300 python tools/standalone_time.py > gpurun_out/w_sa.jsonl 2>&1
MGM_NO_MODE3=1 timeout 300 python tools/standalone_time.py >> gpurun_out/w_sa.jsonl 2>&1
