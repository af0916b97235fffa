mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "gmres or solve or warm or degenerate or full_size_cfg3_vs" > gpurun_out/s_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/s_pytest.log
timeout 900 python tools/ab_solve.py - MGM_NO_MODE3=1 - MGM_NO_MODE3=1 > gpurun_out/s_ab.jsonl 2> gpurun_out/s_ab.err
