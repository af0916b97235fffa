mkdir -p gpurun_out
export MGM_TRACE=1
timeout 600 python tools/ab_solve.py - > gpurun_out/t_ab.jsonl 2> gpurun_out/t_ab.err
cp paper_2204_06154_b200/libmgm_nogather.so paper_2204_06154_b200/libmgm.so
timeout 600 python tools/ab_solve.py - >> gpurun_out/t_ab.jsonl 2>> gpurun_out/t_ab.err
