mkdir -p gpurun_out
MGM_DENSE_BUILD_SINGLE=1 timeout 900 ncu --set full --clock-control none -k regex:k_gs_colour_bs --launch-skip 0 --launch-count 20 \
  -o gpurun_out/batch8_gs2 python tools/batch_trace.py 8 > gpurun_out/b4_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/b4_ncu.log
