cd $GRAFT_REPO_ROOT
cp paper_1607_04808_b200/libfse_b200.so exp/xvar/libfse_b200_base.so
for v in base A B base A B; do
  cp exp/xvar/libfse_b200_$v.so paper_1607_04808_b200/libfse_b200.so
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/x_$v.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/x_$v.json'));print('$v', round(d['ms_per_step'],3),d['stage_ms']['kscale'])"
done
cp exp/xvar/libfse_b200_base.so paper_1607_04808_b200/libfse_b200.so
