mkdir -p gpurun_out
export MGM_TRACE=1
timeout 1200 python tools/ab_solve.py - MGM_L0_VARIANT=1 MGM_L0_VARIANT=2 MGM_L0_VARIANT=3 MGM_L0_VARIANT=1,MGM_GS_BLOCK_L0=128 > gpurun_out/u_ab.jsonl 2> gpurun_out/u_ab.err
