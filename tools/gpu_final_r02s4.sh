# session-4 (HEAD) final state: full GPU suite, smoke, bench as the driver runs it, reference arm, launch list
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/f4_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/f4_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f4_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/f4_smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/f4_bench.json 2> gpurun_out/f4_bench.err
echo "bench rc=$?" >> gpurun_out/f4_bench.err
timeout 900 python bench.py --impl reference --gpus 1 --steps 2 --warmup 1 > gpurun_out/f4_reference.json 2> gpurun_out/f4_reference.err
echo "reference rc=$?" >> gpurun_out/f4_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/f4_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-stages > gpurun_out/f4_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/f4_ncu.log
echo done
