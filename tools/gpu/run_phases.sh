cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_dist.py -q -m gpu -p no:cacheprovider -x 2>&1 | tail -2
timeout 1200 python tools/dist_phases.py cfg2 1 2 4 8 > gpurun_out/dist_phases_cfg2.txt 2>&1; echo rc=$?
timeout 1800 python tools/dist_phases.py cfg5 1 2 4 8 > gpurun_out/dist_phases_cfg5.txt 2>&1; echo rc=$?
tail -5 gpurun_out/dist_phases_cfg2.txt gpurun_out/dist_phases_cfg5.txt
