# FFT v2-kernel mask sweep (FSE_FFT_V2 bits: 1 z fwd, 2 y fwd, 4 x pass, 8 y inv, 16 z inv)
cd $GRAFT_REPO_ROOT
W=${1:-cfg2}; shift
for m in "$@"; do
  FSE_FFT_V2=$m timeout 600 python bench.py --workload $W --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/v2_${W}_$m.json 2>gpurun_out/v2_${W}_$m.err
  python -c "import json;d=json.load(open('gpurun_out/v2_${W}_$m.json'));s=d['stage_ms'];print('$m', round(d['ms_per_step'],3), s['fft_forward'], s['kscale'], s['fft_inverse'])" || tail -3 gpurun_out/v2_${W}_$m.err
done
