# Round-end style measurements: bench lines for every BASELINE workload and the
# tolerance-consistent variants, cfg2 with the CPU baseline, the reference arm
# at cfg2, and the ncu launch list of the default bench.
set -x
cd $GRAFT_REPO_ROOT
TAG=${1:-r02}
for w in cfg1 cfg3 cfg4 cfg5 cfg1t cfg2t cfg3t cfg4t; do
  timeout 900 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_$w.json 2> gpurun_out/${TAG}_bench_$w.err; echo "$w rc=$?"
done
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench_cfg2.json 2> gpurun_out/${TAG}_bench_cfg2.err; echo "cfg2 rc=$?"
timeout 1200 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${TAG}_bench_reference.json 2> gpurun_out/${TAG}_bench_reference.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_ncu_launch.log 2>&1; echo "ncu rc=$?"
