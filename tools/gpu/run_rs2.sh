cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider -k "real or total" > gpurun_out/pytest_rs2.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_rs2.log
for w in cfg2 cfg4; do
timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/brs2_$w.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/brs2_$w.json'));print('$w', round(d['ms_per_step'],3), d['stage_ms']['realspace'])"
done
