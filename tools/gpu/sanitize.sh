cd $GRAFT_REPO_ROOT
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_cfg1.py > gpurun_out/sanitize_$tool.log 2>&1; echo "$tool rc=$?"
  tail -4 gpurun_out/sanitize_$tool.log
done
