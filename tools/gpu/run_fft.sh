cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_fft.py tests/test_gpu_xpass_oracle.py tests/test_gpu_stresslet_engines.py tests/test_gpu_baseline_parity.py tests/test_freespace.py -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_fft.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_fft.log
for w in cfg2 cfg5; do
timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench_$w.json'));print('$w', d['ms_per_step'],d['stage_ms'])"
done
bash tools/gpu/ncu_full.sh r02d "k_xscale2|k_ypass2|k_zfwd2|k_zinv2|k_ypass" 5
