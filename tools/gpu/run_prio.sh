cd $GRAFT_REPO_ROOT
for v in none high low none; do
  if [ $v = none ]; then unset FSE_S1_PRIORITY; else export FSE_S1_PRIORITY=$v; fi
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bprio_$v.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/bprio_$v.json'));print('$v', round(d['ms_per_step'],3))"
  timeout 600 python bench.py --workload cfg4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bprio4_$v.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/bprio4_$v.json'));print('cfg4 $v', round(d['ms_per_step'],3))"
done
