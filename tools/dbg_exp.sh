# development: pass times with parts of the pass disabled (EDAA_DBG bits; results invalid)
for dbg in 0 1 2 3; do echo "EDAA_DBG=$dbg"; EDAA_DBG=$dbg python tools/pass_times.py ${1:-cfg2} 5 2>&1 | tail -1; done
