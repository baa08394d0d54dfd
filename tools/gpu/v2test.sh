cd $GRAFT_REPO_ROOT
for m in -1 31; do
  FSE_FFT_V2=$m timeout 600 python bench.py --workload cfg5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/v2_$m.json 2>gpurun_out/v2_$m.err
  python -c "import json;d=json.load(open('gpurun_out/v2_$m.json'));print('$m', round(d['ms_per_step'],3), {k:round(x,3) for k,x in d['stage_ms'].items()})" || tail -3 gpurun_out/v2_$m.err
done
