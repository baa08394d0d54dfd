cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_dist.py tests/test_cpp_drop_in.py tests/test_cpp_harness.py -q -m gpu -p no:cacheprovider > gpurun_out/pytest_dist.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_dist.log
timeout 600 python bench.py --slabs --steps 5 --warmup 3 > gpurun_out/bench_dist1.json 2> gpurun_out/bench_dist1.err; echo "dist bench rc=$?"
tail -3 gpurun_out/bench_dist1.err
python -c "import json;d=json.load(open('gpurun_out/bench_dist1.json'));print(d['ms_per_step'],d['value'],d['config']['parallelism'])"
