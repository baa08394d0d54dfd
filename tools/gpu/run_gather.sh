cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_gather_paths.py tests/test_gpu_parity.py tests/test_gpu_baseline_parity.py -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_ga.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_ga.log
for w in cfg2 cfg5; do
timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bga_$w.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/bga_$w.json'));print('$w', round(d['ms_per_step'],3), d['stage_ms']['gather'], d['roofline']['kernel'], round(d['roofline']['frac'],3))"
done
