cd $GRAFT_REPO_ROOT
for v in ${DBGS:-0}; do echo "EDAA_DBG=$v"; EDAA_DBG=$v timeout 300 python tools/xp_time.py ${CFGS:-cfg1 cfg2 cfg3} 2>&1 | grep -v f64; done
