# round 2: GPU tests + fused-residual A/B + level-0 colour-kernel ncu (small outputs)
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python tools/ab_solve.py MGM_TRACE=1 MGM_TRACE=1,MGM_NO_FUSE_RR=1 > gpurun_out/ab_fuse.log 2>&1
ARGS="--steps 1 --warmup 3 --no-cpu-baseline --no-stages"
MGM_BENCH_PROFILE=1 python bench.py $ARGS > gpurun_out/plain.log 2>&1
for spec in 'gs|k_gs_colour<\(bool\)0, \(int\)1, \(int\)16, \(bool\)0>|3' 'gszg|k_gs_colour<\(bool\)0, \(int\)1, \(int\)16, \(bool\)1>|2' 'rr|k_res_restrict|2'; do
  IFS='|' read -r tag pat cnt <<< "$spec"
  MGM_BENCH_PROFILE=1 ncu --profile-from-start off --set full --clock-control none --import-source on \
     --kernel-name-base demangled -k "regex:$pat" -c $cnt -o gpurun_out/r02_$tag python bench.py $ARGS > gpurun_out/ncu_$tag.log 2>&1
  ncu -i gpurun_out/r02_$tag.ncu-rep --page raw --csv > gpurun_out/r02_${tag}_raw.csv 2>&1
  ncu -i gpurun_out/r02_$tag.ncu-rep --page details --csv > gpurun_out/r02_${tag}_details.csv 2>&1
  ncu -i gpurun_out/r02_$tag.ncu-rep --page source --csv > gpurun_out/r02_${tag}_source.csv 2>&1
  rm -f gpurun_out/r02_$tag.ncu-rep
done
MGM_SETUP_TIMING=1 python tools/ab_solve.py - > gpurun_out/setup_timing.log 2>&1
echo done
