cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden.py -q -m gpu -p no:cacheprovider -k "spread or total" > gpurun_out/pytest_sp.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_sp.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bsp.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/bsp.json'));print(round(d['ms_per_step'],3), d['stage_ms']['spread'])"
