# ncu --set full of the step's hot kernels at cfg2 (one launch each), with source;
# exports CSV pages on the box and keeps the .ncu-rep only if small
cd $GRAFT_REPO_ROOT
TAG=${1:-r02a}
KR=${2:-"k_xscale2|k_realspace|k_gather_tma|k_spread|k_ypass2|k_zfwd2|k_zinv2|k_ypass"}
CNT=${3:-9}
timeout 900 python tools/profile_step.py cfg2 1 > gpurun_out/prof_${TAG}_plain.log 2>&1; echo "plain rc=$?"
FSE_SERIAL=1 timeout 1500 ncu --set full --import-source on --clock-control none \
  -k "regex:${KR}" -c ${CNT} -o /tmp/prof_${TAG} -f \
  python tools/profile_step.py cfg2 1 > gpurun_out/prof_${TAG}.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/prof_${TAG}.log
ncu -i /tmp/prof_${TAG}.ncu-rep --page raw --csv > gpurun_out/prof_${TAG}_raw.csv 2>/dev/null
python tools/ncu_summary.py full /tmp/prof_${TAG}.ncu-rep > gpurun_out/prof_${TAG}_summary.md 2>&1
for k in $(echo $KR | tr '|' ' '); do
  ncu -i /tmp/prof_${TAG}.ncu-rep --page source --csv -k "regex:$k" --print-source sass \
    > gpurun_out/prof_${TAG}_src_${k}.csv 2>/dev/null
done
ls -la gpurun_out/ | head -40
du -sh gpurun_out
