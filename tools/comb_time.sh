# warm per-launch durations of the between-pass kernels (dev): bash tools/comb_time.sh cfg1
cd $GRAFT_REPO_ROOT
c=${1:-cfg1}
EDAA_NO_GRAPH=1 python tools/prof_solve.py $c 1 > /dev/null 2>&1
EDAA_NO_GRAPH=1 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv \
  --log-file gpurun_out/comb_$c.csv python tools/prof_solve.py $c 1 > /dev/null 2>&1
python tools/launches.py gpurun_out/comb_$c.csv | head -14
