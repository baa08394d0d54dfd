# A/B of CTA-shared real-space kernel variants (exp/<v>/libfse_b200.so), forced with FSE_RS_WARP=0
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_realspace_kernels.py -q -x -p no:cacheprovider 2>&1 | tail -4
for v in "$@"; do
  for w in cfg2 cfg4; do
    FSE_RS_WARP=0 FSE_LIB_PATH=$GRAFT_REPO_ROOT/exp/$v/libfse_b200.so timeout 600 python bench.py --workload $w --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/rsc.json 2> gpurun_out/rsc.err
    python -c "import json;d=json.load(open('gpurun_out/rsc.json'));print('$v $w', round(d['ms_per_step'],3), round(d['stage_ms']['realspace'],3))" || tail -3 gpurun_out/rsc.err
  done
done
