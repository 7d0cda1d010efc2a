for dbg in 3 7 11 19 35 63; do echo "EDAA_DBG=$dbg"; EDAA_DBG=$dbg python tools/pass_times.py ${1:-cfg2} 5 2>&1 | tail -1; done
