# ncu --set full of one kernel launch at cfg2 with source views (sass + cuda lines)
cd $GRAFT_REPO_ROOT
TAG=$1; K=$2; W=${3:-cfg2}
FSE_SERIAL=1 timeout 900 ncu --set full --import-source on --clock-control none \
  -k "regex:${K}" -c 1 -o /tmp/prof_${TAG} -f python tools/profile_step.py $W 1 > gpurun_out/prof_${TAG}.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py full /tmp/prof_${TAG}.ncu-rep > gpurun_out/prof_${TAG}_summary.md 2>&1
ncu -i /tmp/prof_${TAG}.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_${TAG}_sass.csv 2>/dev/null
ncu -i /tmp/prof_${TAG}.ncu-rep --page source --csv --print-source cuda > gpurun_out/prof_${TAG}_cuda.csv 2>/dev/null
ncu -i /tmp/prof_${TAG}.ncu-rep --page details --csv > gpurun_out/prof_${TAG}_details.csv 2>/dev/null
ls -la gpurun_out/prof_${TAG}*
