# round-2 final-state evidence (after the multi-RHS and device-LU changes)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/fe_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/fe_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fe_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/fe_smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/fe_bench.json 2> gpurun_out/fe_bench.err
echo "bench rc=$?" >> gpurun_out/fe_bench.err
ARGS="--steps 1 --warmup 3 --no-cpu-baseline --no-stages"
MGM_BENCH_PROFILE=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/fe_launches.csv python bench.py $ARGS > gpurun_out/fe_ncu_l.log 2>&1
MGM_DENSE_BUILD_SINGLE=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gs_colour_bs \
  --launch-skip 16 --launch-count 2 -o gpurun_out/fe_batch8 python tools/batch_trace.py 8 > gpurun_out/fe_ncu_b8.log 2>&1
ncu -i gpurun_out/fe_batch8.ncu-rep --page details --csv > gpurun_out/fe_batch8_details.csv 2>&1
rm -f gpurun_out/fe_batch8.ncu-rep
: > gpurun_out/fe_all_configs.jsonl
for args in "--cfg 1" "--cfg 2" "--cfg 2 --method gfd" "--cfg 4 --n 262144" "--cfg 5"; do
  timeout 1500 python bench.py $args --steps 3 --warmup 3 --no-cpu-baseline --no-stages > gpurun_out/ac.out 2> gpurun_out/ac.err
  echo "{\"args\": \"$args\", \"rc\": $?}" >> gpurun_out/fe_all_configs.jsonl
  tail -1 gpurun_out/ac.out >> gpurun_out/fe_all_configs.jsonl
done
echo done
