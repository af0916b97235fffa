# ncu launch list of the bench's timed region with the host-loop GMRES (same kernels; the device
# GMRES's WHILE-node graph cannot be profiled by ncu), plus the plain run for comparison
mkdir -p gpurun_out
ARGS="--steps 1 --warmup 3 --no-cpu-baseline --no-stages"
MGM_HOST_GMRES=1 timeout 600 python bench.py $ARGS > gpurun_out/ll_plain.json 2> gpurun_out/ll_plain.err
MGM_HOST_GMRES=1 MGM_BENCH_PROFILE=1 timeout 1200 ncu --profile-from-start off --metrics gpu__time_duration.sum \
  --clock-control none --csv --log-file gpurun_out/ll_launches.csv python bench.py $ARGS > gpurun_out/ll_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/ll_ncu.log
