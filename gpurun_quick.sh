cd $GRAFT_REPO_ROOT
nproc; free -g | head -2; lscpu | grep -E "Model name|Socket|Core|Thread" 
python -c "import __graft_entry__ as g; g.smoke()"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu 2>&1 | tail -5
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo bench rc=$?
cat gpurun_out/bench_cfg2.json; tail -5 gpurun_out/bench_cfg2.err
