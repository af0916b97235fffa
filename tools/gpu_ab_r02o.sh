mkdir -p gpurun_out
export MGM_TRACE=1
timeout 1200 python tools/ab_solve.py - MGM_GS_BLOCK_L0=128 MGM_GS_BLOCK_L0=64 MGM_GS_BLOCK_L0=512 MGM_L0_TPR=2,MGM_GS_BLOCK_L0=128 > gpurun_out/o_ab.jsonl 2> gpurun_out/o_ab.err
