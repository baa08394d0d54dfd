cd $GRAFT_REPO_ROOT
for w in cfg3 cfg4; do
  FSE_SERIAL=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_realspace -c 1 -o /tmp/rs_$w -f python tools/profile_step.py $w 0 > gpurun_out/rs_calib_$w.log 2>&1
  ncu -i /tmp/rs_$w.ncu-rep --page source --csv --print-source sass > gpurun_out/rs_calib_${w}_src.csv 2>/dev/null
  python tools/ncu_summary.py full /tmp/rs_$w.ncu-rep > gpurun_out/rs_calib_${w}_summary.md 2>&1
  timeout 600 python bench.py --workload $w --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/rs_calib_${w}.json 2>/dev/null
done
