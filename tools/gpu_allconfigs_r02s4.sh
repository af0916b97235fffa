# session-4 (HEAD): every BASELINE config through bench.py (setup times with the GPU WSE + GPU iterated-greedy passes)
mkdir -p gpurun_out
: > gpurun_out/f4_all_configs.jsonl
for args in "--cfg 1" "--cfg 2" "--cfg 2 --method gfd" "--cfg 4 --n 262144" "--cfg 4" "--cfg 5"; do
  timeout 1500 python bench.py $args --steps 3 --warmup 3 --no-cpu-baseline --no-stages > gpurun_out/ac.out 2> gpurun_out/ac.err
  echo "{\"args\": \"$args\", \"rc\": $?}" >> gpurun_out/f4_all_configs.jsonl
  tail -1 gpurun_out/ac.out >> gpurun_out/f4_all_configs.jsonl
done
echo done
