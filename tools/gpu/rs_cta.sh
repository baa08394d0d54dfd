# CTA-shared real-space kernel: parity tests, then A/B against the warp-item kernel
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge_cases.py tests/test_gpu_baseline_parity.py tests/test_gpu_dist.py -q -x -p no:cacheprovider 2>&1 | tail -6
for w in cfg2 cfg4 cfg3 cfg1; do
  for e in 0 1; do
    FSE_RS_WARP=$e timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/rs_$w_$e.json 2> gpurun_out/rs_$w_$e.err
    python -c "import json;d=json.load(open('gpurun_out/rs_$w_$e.json'));print('$w warp=$e', round(d['ms_per_step'],3), {k:round(x,3) for k,x in d['stage_ms'].items() if k in ('realspace','realspace_binning','call')})" || tail -3 gpurun_out/rs_$w_$e.err
  done
done
