mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "standalone or solve or warm or degenerate or gmres or dist_fake" > gpurun_out/x_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/x_pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-stages > gpurun_out/x_bench.json 2> gpurun_out/x_bench.err
MGM_NO_MODE3=1 timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-stages > gpurun_out/x_bench0.json 2>> gpurun_out/x_bench.err
