mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "device_coarse_lu or per_operator or dense_bottom or error" > gpurun_out/l_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/l_pytest.log
timeout 900 python tools/setup_timing.py 5 > gpurun_out/l_setup5.txt 2>&1
echo "rc=$?" >> gpurun_out/l_setup5.txt
