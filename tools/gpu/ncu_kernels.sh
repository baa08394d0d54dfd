# ncu --set full of every step kernel at cfg2 (one launch each), summary table
# and dram bytes per kernel (profiles/traffic.json)
cd $GRAFT_REPO_ROOT
TAG=${1:-s2}
KR="k_spread_ws|k_gather_tma|k_xscale2|k_realspace|k_ypass|k_zfwd2|k_zinv2|k_payload"
FSE_SERIAL=1 timeout 1500 ncu --set full --import-source on --clock-control none \
  -k "regex:${KR}" -c 8 -o /tmp/prof_${TAG} -f \
  python tools/profile_step.py cfg2 1 > gpurun_out/prof_${TAG}.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py full /tmp/prof_${TAG}.ncu-rep > gpurun_out/prof_${TAG}_summary.md 2>&1
ncu -i /tmp/prof_${TAG}.ncu-rep --page raw --csv > gpurun_out/prof_${TAG}_raw.csv 2>/dev/null
for k in k_spread_ws k_gather_tma k_xscale2 k_realspace; do
  ncu -i /tmp/prof_${TAG}.ncu-rep --page source --csv --print-source sass -k "regex:$k" > gpurun_out/prof_${TAG}_sass_$k.csv 2>/dev/null
done
cat gpurun_out/prof_${TAG}_summary.md
