# round 2: batched V-cycle launch list; in-situ DRAM bytes of the solve's kernels (application
# replay, caches not flushed)
set -x
mkdir -p gpurun_out
python tools/batch_profile.py 8 > gpurun_out/batch8.log 2>&1 && \
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r02_batch8_launches.csv python tools/batch_profile.py 8 > gpurun_out/ncu_b8.log 2>&1
ARGS="--steps 1 --warmup 3 --no-cpu-baseline --no-stages"
MGM_BENCH_PROFILE=1 python bench.py $ARGS > gpurun_out/plain.log 2>&1 && \
MGM_BENCH_PROFILE=1 ncu --profile-from-start off --cache-control none --replay-mode application \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/r02_insitu_dram.csv python bench.py $ARGS > gpurun_out/ncu_insitu.log 2>&1
echo done
python tools/ab_solve.py --cfg 5 --n 4194304 MGM_TRACE=1 MGM_TRACE=1,MGM_NO_FUSE_RR=1 > gpurun_out/ab_cfg5_4m.log 2>&1
echo done2
