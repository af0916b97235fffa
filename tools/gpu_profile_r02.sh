# bench + ncu evidence for round 2 (one gpurun call; outputs kept small: CSV exports, reports removed)
set -x
mkdir -p gpurun_out
python bench.py --steps 5 --warmup 3 > gpurun_out/bench2.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench2.log
ARGS="--steps 1 --warmup 3 --no-cpu-baseline --no-stages"
MGM_BENCH_PROFILE=1 python bench.py $ARGS > gpurun_out/plain.log 2>&1 && \
MGM_BENCH_PROFILE=1 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv python bench.py $ARGS > gpurun_out/ncu_l.log 2>&1
for spec in "gs|k_gs_colour<false, 1, 16, false>|3" "gszg|k_gs_colour<false, 1, 16, true>|2" "dense|k_dense_apply|1" "spmv|k_sell_spmv|3" "interp|k_interp_correct|1"; do
  IFS='|' read -r tag pat cnt <<< "$spec"
  MGM_BENCH_PROFILE=1 ncu --profile-from-start off --set full --clock-control none --import-source on \
     --kernel-name-base demangled -k "regex:$pat" -c $cnt -o gpurun_out/r02_$tag python bench.py $ARGS > gpurun_out/ncu_$tag.log 2>&1
  ncu -i gpurun_out/r02_$tag.ncu-rep --page raw --csv > gpurun_out/r02_${tag}_raw.csv 2>&1
  ncu -i gpurun_out/r02_$tag.ncu-rep --page details --csv > gpurun_out/r02_${tag}_details.csv 2>&1
  rm -f gpurun_out/r02_$tag.ncu-rep
done
ls -la gpurun_out
echo done
