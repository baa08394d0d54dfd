cd $GRAFT_REPO_ROOT
for t in 160 320 640 1280 2560; do
  for w in cfg4 cfg3; do
    FSE_RS_OCT=$t timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/rso.json 2> gpurun_out/rso.err
    python -c "import json;d=json.load(open('gpurun_out/rso.json'));print('OCT=$t $w', round(d['ms_per_step'],3), round(d['stage_ms']['realspace'],3))" || tail -3 gpurun_out/rso.err
  done
done
