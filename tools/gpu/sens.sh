cd $GRAFT_REPO_ROOT
timeout 1200 python tools/green_sensitivity.py 2>&1 | tee gpurun_out/sens.log
