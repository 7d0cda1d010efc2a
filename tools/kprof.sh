# Per-phase cycle accounting (EDAA_KPROF=1) and pass times under development switches.
# usage: tools/kprof2.sh cfg1 "0 256 1 128"
c=${1:-cfg1}
for dbg in ${2:-0}; do
  echo "== $c EDAA_DBG=$dbg"
  EDAA_DBG=$dbg EDAA_KPROF=1 python tools/prof_solve.py $c 1 2>&1 | grep -E "kprof\] +(A|B)"
  EDAA_DBG=$dbg python tools/pass_times.py $c 3 2>&1 | tail -1
done
