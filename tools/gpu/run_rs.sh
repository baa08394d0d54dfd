cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_parity.py -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_rs.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_rs.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench_cfg2.json'));print(d['ms_per_step'],d['stage_ms'])"
timeout 600 python bench.py --workload cfg4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo "bench4 rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench_cfg4.json'));print(d['ms_per_step'],d['stage_ms'])"
bash tools/gpu/ncu_full.sh r02c "k_realspace" 1
