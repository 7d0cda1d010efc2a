for dbg in 0 2 66 130 194; do echo "EDAA_DBG=$dbg"; EDAA_DBG=$dbg python tools/pass_times.py ${1:-cfg2} 3 2>&1 | tail -1; done
