# device iterated-greedy colouring passes: parity, full-size cfg3 parity, setup timing cfg3/cfg5
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "device_colouring or structures or full_size_cfg3_vs_oracle or device_wse" > gpurun_out/ig_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/ig_pytest.log
for c in 3 5; do timeout 900 bash tools/setup_timing.sh $c; mv gpurun_out/setup_timing_cfg$c.log gpurun_out/ig_cfg$c.log; done
echo done
