# Round profiling bundle (run on the GPU box).  part 1: bench line + launch lists;
# part 2: one full ncu capture of the B pass and of the A pass (cfg given).
part=${1:-1}; c=${2:-cfg1}
if [ "$part" = 1 ]; then
  python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
  for c in cfg1 cfg2; do
    EDAA_NO_GRAPH=1 python tools/prof_solve.py $c 1 > gpurun_out/plain_$c.log 2>&1 && \
    EDAA_NO_GRAPH=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/launches_$c.csv python tools/prof_solve.py $c 1 > gpurun_out/ncu_l_$c.log 2>&1
  done
  cat gpurun_out/bench_default.json
else
  EDAA_NO_GRAPH=1 python tools/prof_solve.py $c 1 > gpurun_out/plain_$c.log 2>&1 && \
  EDAA_NO_GRAPH=1 ncu --set full --clock-control none --import-source on -k regex:k_pass -s 2 -c 1 \
      -o gpurun_out/full_B_$c python tools/prof_solve.py $c 1 > gpurun_out/ncu_f_$c.log 2>&1
  EDAA_NO_GRAPH=1 ncu --set full --clock-control none -k regex:k_pass -s 1 -c 1 \
      -o gpurun_out/full_A_$c python tools/prof_solve.py $c 1 > gpurun_out/ncu_fa_$c.log 2>&1
  for r in full_B_$c full_A_$c; do
    ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv 2>/dev/null
    ncu -i gpurun_out/$r.ncu-rep --page details --csv > gpurun_out/${r}_details.csv 2>/dev/null
  done
  rm -f gpurun_out/full_A_$c.ncu-rep
  # launch list of the bench command itself (first 400 launches)
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file gpurun_out/launches_bench.csv python bench.py --steps 1 --warmup 3 > gpurun_out/ncu_bench.log 2>&1
  ls -la gpurun_out/
fi
