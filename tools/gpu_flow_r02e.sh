# flow sweep: parity tests, then A/B on cfg3
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "flow" > gpurun_out/f_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/f_pytest.log
export MGM_TRACE=1
timeout 1200 python tools/ab_solve.py MGM_FLOW=0 - MGM_FLOW_PF=0 MGM_FLOW_CPS=1 MGM_FLOW_MIN=60000 MGM_FLOW_MIN=0 > gpurun_out/f_ab.jsonl 2> gpurun_out/f_ab.err
echo "ab rc=$?" >> gpurun_out/f_ab.err
