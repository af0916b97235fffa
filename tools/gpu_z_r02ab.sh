mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -k "solve or warm or degenerate or gmres or full_size or dist or poisson" > gpurun_out/ab_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/ab_pytest.log
