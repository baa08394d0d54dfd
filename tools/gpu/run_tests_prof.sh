set -x
cd $GRAFT_REPO_ROOT
export FSE_PARITY_LOG=$GRAFT_REPO_ROOT/gpurun_out/parity_r02.jsonl
rm -f $FSE_PARITY_LOG
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log
bash tools/gpu/ncu_full.sh r02a
