# per-phase cycle accounting of the pass kernels (EDAA_KPROF=1), cfg2 T=1
for c in cfg2 cfg1; do EDAA_KPROF=1 python tools/prof_solve.py $c 1 2>&1 | tail -3; done
