cd $GRAFT_REPO_ROOT
cp paper_1607_04808_b200/libfse_b200.so /tmp/orig.so
for mb in 2 3 4; do
  cp exp/rsvar/libfse_b200_$mb.so paper_1607_04808_b200/libfse_b200.so
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/rs_$mb.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/rs_$mb.json'));print($mb, d['ms_per_step'],d['stage_ms']['realspace'])"
  timeout 600 python bench.py --workload cfg4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/rs4_$mb.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/rs4_$mb.json'));print('cfg4',$mb, d['ms_per_step'],d['stage_ms']['realspace'])"
done
cp /tmp/orig.so paper_1607_04808_b200/libfse_b200.so
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider -x -k "real or total" 2>&1 | tail -2
