mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "solve or warm or degenerate or gmres or full_size" > gpurun_out/aa_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/aa_pytest.log
timeout 900 python tools/ab_solve.py - MGM_GMRES_NO_Z=1 - > gpurun_out/aa_ab.jsonl 2> gpurun_out/aa_ab.err
