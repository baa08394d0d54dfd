# A/B timing of library variants: bash tools/gpu/ab.sh WORKLOAD lib1 lib2 ...
cd $GRAFT_REPO_ROOT
W=$1; shift
for v in "$@"; do
  for rep in 1 2; do
    FSE_LIB_PATH=$GRAFT_REPO_ROOT/exp/$v/libfse_b200.so timeout 600 python bench.py --workload $W --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab_${W}_${v}_$rep.json 2> gpurun_out/ab_${W}_${v}_$rep.err
    python -c "import json,sys;d=json.load(open('gpurun_out/ab_${W}_${v}_$rep.json'));print('$v', '$rep', round(d['ms_per_step'],3), {k:round(x,3) for k,x in d['stage_ms'].items()})" || tail -3 gpurun_out/ab_${W}_${v}_$rep.err
  done
done
