# setup stage timings after the colouring changes (cfg3, cfg5)
mkdir -p gpurun_out
for c in 3 5; do timeout 900 bash tools/setup_timing.sh $c; mv gpurun_out/setup_timing_cfg$c.log gpurun_out/s3col_cfg$c.log; done
echo done
