mkdir -p gpurun_out
export MGM_TRACE=1
timeout 900 python tools/ab_solve.py MGM_L0_TPR=2 MGM_L0_TPR=2,MGM_FLOW=0 MGM_L0_TPR=4 MGM_L0_TPR=2,MGM_FLOW_PF=0 > gpurun_out/f2_ab.jsonl 2> gpurun_out/f2_ab.err
