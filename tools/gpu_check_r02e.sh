# re-entry check: GPU tests + bench at the restored state
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/e_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/e_pytest.log
timeout 600 python bench.py --gpus 1 --steps 10 --warmup 3 > gpurun_out/e_bench.json 2> gpurun_out/e_bench.err
echo "bench rc=$?" >> gpurun_out/e_bench.err
