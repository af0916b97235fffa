mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "batch" > gpurun_out/z_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/z_pytest.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/z_bench.json 2> gpurun_out/z_bench.err
