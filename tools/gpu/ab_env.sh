# A/B of one library under environment settings: bash tools/gpu/ab_env.sh WORKLOAD LIB "ENV1" "ENV2" ...
cd $GRAFT_REPO_ROOT
W=$1; V=$2; shift 2
for e in "$@"; do
  env $e FSE_LIB_PATH=$GRAFT_REPO_ROOT/exp/$V/libfse_b200.so timeout 600 python bench.py --workload $W --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/abe.json 2> gpurun_out/abe.err
  python -c "import json;d=json.load(open('gpurun_out/abe.json'));print('$e', round(d['ms_per_step'],3), {k:round(x,3) for k,x in d['stage_ms'].items()})" || tail -3 gpurun_out/abe.err
done
