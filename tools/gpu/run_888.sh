cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_fft.py tests/test_gpu_xpass_oracle.py -q -m gpu -p no:cacheprovider > gpurun_out/pytest_888.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_888.log
timeout 900 python bench.py --workload cfg2t --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_cfg2t.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/r02_bench_cfg2t.json'));c=d['config'];print('cfg2t', round(d['ms_per_step'],2), '%.3g'%d['value'], {k:round(v,2) for k,v in d['stage_ms'].items()})"
