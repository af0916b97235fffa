# round-2 session-3 re-entry check: full GPU suite, smoke, bench at the restored commit
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/s3_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/s3_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/s3_smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/s3_bench.json 2> gpurun_out/s3_bench.err
echo "bench rc=$?" >> gpurun_out/s3_bench.err
echo done
