mkdir -p gpurun_out
export MGM_TRACE=1
timeout 1200 python tools/ab_solve.py - MGM_LJ_TPR=8 MGM_LJ_TPR=2 MGM_GS_BLOCK_SMALL=128 MGM_GS_BLOCK_SMALL=256 > gpurun_out/n_ab.jsonl 2> gpurun_out/n_ab.err
