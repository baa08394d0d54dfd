# ncu --set full of the step's hot kernels at cfg2 (one launch each), with source
cd $GRAFT_REPO_ROOT
TAG=${1:-r02a}
KR=${2:-"k_xscale2|k_realspace|k_gather_tma|k_spread|k_ypass2|k_zfwd2|k_zinv2|k_ypass"}
timeout 900 python tools/profile_step.py cfg2 1 > gpurun_out/prof_${TAG}_plain.log 2>&1; echo "plain rc=$?"
FSE_SERIAL=1 timeout 1500 ncu --set full --import-source on --clock-control none \
  -k "regex:${KR}" -c 9 -o gpurun_out/prof_${TAG} -f \
  python tools/profile_step.py cfg2 1 > gpurun_out/prof_${TAG}.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/prof_${TAG}.log
