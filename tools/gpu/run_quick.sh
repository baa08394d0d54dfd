set -x
cd $GRAFT_REPO_ROOT
export FSE_PARITY_LOG=$GRAFT_REPO_ROOT/gpurun_out/parity_r02.jsonl
rm -f $FSE_PARITY_LOG
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench_cfg2.json'));print(d['ms_per_step'],d['stage_ms'])"
bash tools/gpu/ncu_full.sh r02b "k_xscale2|k_realspace" 2
