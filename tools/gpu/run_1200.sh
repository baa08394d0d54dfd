cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_fft.py tests/test_gpu_xpass_oracle.py tests/test_gpu_stresslet_engines.py -q -m gpu -p no:cacheprovider > gpurun_out/pytest_1200.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_1200.log
for v in 3l 2l; do
  if [ $v = 2l ]; then export FSE_FFT_1200_2L=1; fi
  timeout 600 python bench.py --workload cfg5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b1200_$v.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/b1200_$v.json'));print('$v', d['ms_per_step'],{k:round(x,2) for k,x in d['stage_ms'].items()})"
done
