# round 2 final-state evidence: driver-like bench, reference arm, smoke, every config
mkdir -p gpurun_out
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
echo "bench rc=$?" >> gpurun_out/final_bench.err
python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err
echo "ref rc=$?" >> gpurun_out/final_ref.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/final_smoke.log
bash tools/gpu_allconfigs_r02.sh
echo done
