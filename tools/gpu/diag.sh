cd $GRAFT_REPO_ROOT
timeout 1200 python tools/parity_diag.py cfg1 cfg2s cfg2 2>&1 | tee gpurun_out/diag.log
