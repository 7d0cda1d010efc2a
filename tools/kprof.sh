# per-phase cycle accounting of the pass kernels (EDAA_KPROF=1), T=1 solve
for c in ${1:-cfg2}; do for dbg in 0 2; do echo "$c EDAA_DBG=$dbg"; EDAA_DBG=$dbg EDAA_KPROF=1 python tools/prof_solve.py $c 1 2>&1 | grep -E "kprof\] +(A|B)"; done; done
