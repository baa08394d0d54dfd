cd $GRAFT_REPO_ROOT
for v in 2l 3l; do
  if [ $v = 3l ]; then export FSE_FFT_624_3L=1; fi
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b624_$v.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/b624_$v.json'));print('$v', d['ms_per_step'],{k:round(x,2) for k,x in d['stage_ms'].items()})"
done
FSE_FFT_624_3L=1 timeout 600 python -m pytest tests/test_gpu_fft.py -q -m gpu -p no:cacheprovider -k "624" 2>&1 | tail -2
