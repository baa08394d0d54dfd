# real space: octant items of dense cells (FSE_RS_OCT = threshold, 0 = off)
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge_cases.py tests/test_gpu_realspace_kernels.py -q -x -p no:cacheprovider 2>&1 | tail -12
FSE_RS_OCT=32 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_realspace_kernels.py tests/test_gpu_baseline_parity.py -q -x -p no:cacheprovider 2>&1 | tail -12
for t in "$@"; do
  for w in cfg4 cfg3 cfg2 cfg5 cfg1; do
    FSE_RS_OCT=$t timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/rso.json 2> gpurun_out/rso.err
    python -c "import json;d=json.load(open('gpurun_out/rso.json'));print('OCT=$t $w', round(d['ms_per_step'],3), round(d['stage_ms']['realspace'],3), round(d['stage_ms']['realspace_binning'],3))" || tail -3 gpurun_out/rso.err
  done
done
