# persisting-L2 window over the level-0 iterate (MGM_L2_WIN=MB) vs none: traced V-cycle + solve
mkdir -p gpurun_out
timeout 1200 python tools/ab_solve.py - MGM_L2_WIN=16 MGM_L2_WIN=40 - > gpurun_out/l2win.jsonl 2> gpurun_out/l2win.err
echo "rc=$?" >> gpurun_out/l2win.err
