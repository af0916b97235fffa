# device WSE: parity tests, then setup timing (device vs host WSE) on cfg3 and cfg5
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "device_wse or device_knn or error_paths or structures" > gpurun_out/wse_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/wse_pytest.log
for c in 3 5; do
  timeout 900 bash tools/setup_timing.sh $c; mv gpurun_out/setup_timing_cfg$c.log gpurun_out/wse_dev_cfg$c.log
  MGM_HOST_WSE=1 timeout 900 bash tools/setup_timing.sh $c; mv gpurun_out/setup_timing_cfg$c.log gpurun_out/wse_host_cfg$c.log
done
echo done
