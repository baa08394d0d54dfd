cd $GRAFT_REPO_ROOT
export FSE_PARITY_LOG=$GRAFT_REPO_ROOT/gpurun_out/parity_r02.jsonl
rm -f $FSE_PARITY_LOG
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider -s > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
grep "cfg2t rel rms" gpurun_out/pytest_gpu.log
for w in cfg1t cfg2t cfg3t cfg4t; do
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_$w.json 2> gpurun_out/r02_bench_$w.err; echo "$w rc=$?"
  python -c "import json;d=json.load(open('gpurun_out/r02_bench_$w.json'));c=d['config'];print('$w', round(d['ms_per_step'],2), '%.3g'%d['value'], c['M'], c['fft_grid'], {k:round(v,2) for k,v in d['stage_ms'].items()})"
done
