set -x
cd $GRAFT_REPO_ROOT
nproc; free -g | head -2; lscpu | grep "Model name"
export FSE_PARITY_LOG=$GRAFT_REPO_ROOT/gpurun_out/parity_r02.jsonl
rm -f $FSE_PARITY_LOG
timeout 1500 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo "bench rc=$?"
cat gpurun_out/bench_cfg2.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
cat gpurun_out/bench_ref.json
