# Round-end run: the whole GPU test suite, bench lines of every workload (incl.
# cfg5t), the default bench with the CPU baseline, the reference arm, and the ncu
# launch list of the default bench.  bash tools/gpu/round_end.sh [TAG]
set -x
cd $GRAFT_REPO_ROOT
TAG=${1:-r02e}
export FSE_PARITY_LOG=$GRAFT_REPO_ROOT/gpurun_out/${TAG}_parity.jsonl
rm -f $FSE_PARITY_LOG
timeout 1800 python -m pytest tests -q -m gpu -x -p no:cacheprovider --durations=8 > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -14 gpurun_out/${TAG}_pytest_gpu.log
unset FSE_PARITY_LOG
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${TAG}_smoke.log
for w in cfg1 cfg3 cfg4 cfg5 cfg1t cfg2t cfg3t cfg4t; do
  timeout 900 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_$w.json 2> gpurun_out/${TAG}_bench_$w.err; echo "$w rc=$?"
done
timeout 900 python bench.py --workload cfg5t --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_cfg5t.json 2> gpurun_out/${TAG}_bench_cfg5t.err; echo "cfg5t rc=$?"
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench_cfg2.json 2> gpurun_out/${TAG}_bench_cfg2.err; echo "cfg2 rc=$?"
timeout 1200 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_bench_reference.json 2> gpurun_out/${TAG}_bench_reference.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_ncu_launch.log 2>&1; echo "ncu rc=$?"
for f in gpurun_out/${TAG}_bench_*.json; do python -c "
import json,sys
d=json.load(open('$f')); print('$f', round(d['ms_per_step'],3), d['value'], d.get('e2e',{}).get('value'), d.get('roofline',{}).get('frac'))" || tail -2 ${f%.json}.err; done
