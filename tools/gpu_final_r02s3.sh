# session-3 final state: full GPU suite, smoke, bench, all configs (setup times incl. GPU WSE)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/f3_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/f3_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f3_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/f3_smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/f3_bench.json 2> gpurun_out/f3_bench.err
echo "bench rc=$?" >> gpurun_out/f3_bench.err
: > gpurun_out/f3_all_configs.jsonl
for args in "--cfg 1" "--cfg 2" "--cfg 2 --method gfd" "--cfg 4 --n 262144" "--cfg 5"; do
  timeout 1500 python bench.py $args --steps 3 --warmup 3 --no-cpu-baseline --no-stages > gpurun_out/ac.out 2> gpurun_out/ac.err
  echo "{\"args\": \"$args\", \"rc\": $?}" >> gpurun_out/f3_all_configs.jsonl
  tail -1 gpurun_out/ac.out >> gpurun_out/f3_all_configs.jsonl
done
echo done
