# A/B timing of the split MMA roles vs the unified assignment (dev)
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
timeout 300 python tools/xp_time.py ${CFGS:-cfg1 cfg2 cfg3} 2>&1 | grep -v f64
echo "--- EDAA_NO_SPLIT=1"
EDAA_NO_SPLIT=1 timeout 300 python tools/xp_time.py ${CFGS:-cfg1 cfg2 cfg3} 2>&1 | grep -v f64
