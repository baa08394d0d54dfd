cd $GRAFT_REPO_ROOT
export FSE_PHASES_VERBOSE=1
timeout 1200 python tools/dist_phases.py cfg2 1 2 > gpurun_out/dp2.txt 2>&1; echo rc=$?
timeout 1800 python tools/dist_phases.py cfg5 8 > gpurun_out/dp5.txt 2>&1; echo rc=$?
cat > /tmp/one.py <<'PY'
import sys, os
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"])
import numpy as np, bench, paper_1607_04808_b200 as fse
ctx = fse.Context(0)
w = bench.WORKLOADS["cfg2"]
s, _ = fse.generate_workload(1, w["n"], bench.SEED)
cfg = fse.make_config(1.0, 110., 0.045, 288, 24)
g = ctx.precompute_mollified_green(1, cfg.Ltilde, cfg.Mtilde, cfg.sf)
ctx.dist_virtual_total_sum(s, 0, cfg, s.positions, g, 1, targets_are_sources=True)
ctx.dist_virtual_total_sum(s, 0, cfg, s.positions, g, 1, targets_are_sources=True)
PY
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/dp_launch.csv python /tmp/one.py > /dev/null 2>&1; echo ncu=$?
python tools/ncu_summary.py launches gpurun_out/dp_launch.csv > gpurun_out/dp_launch.md
head -25 gpurun_out/dp_launch.md
