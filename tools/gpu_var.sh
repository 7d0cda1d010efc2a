cd $GRAFT_REPO_ROOT
for v in ${VARS}; do echo "VAR=$v"; EDAA_CUDA_LIB=$PWD/paper_2209_11002_b200/$v EDAA_DBG=${DBG:-0} timeout 300 python tools/xp_time.py ${CFGS:-cfg1 cfg2} 2>&1 | grep -v f64; done
