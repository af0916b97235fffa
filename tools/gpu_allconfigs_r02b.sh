# every BASELINE config through bench.py (one B200), one JSON line each -> gpurun_out/r02b_all_configs.jsonl
mkdir -p gpurun_out
: > gpurun_out/r02b_all_configs.jsonl
for args in "--cfg 1" "--cfg 2" "--cfg 2 --method gfd" "--cfg 4 --n 262144" "--cfg 5"; do
  timeout 1500 python bench.py $args --steps 3 --warmup 3 --no-cpu-baseline --no-stages > gpurun_out/ac.out 2> gpurun_out/ac.err
  echo "{\"args\": \"$args\", \"rc\": $?}" >> gpurun_out/r02b_all_configs.jsonl
  tail -1 gpurun_out/ac.out >> gpurun_out/r02b_all_configs.jsonl
  tail -3 gpurun_out/ac.err >> gpurun_out/r02b_all_configs_err.txt
done
