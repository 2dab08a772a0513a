cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  for c in c1 c3 corners stream small tc er formats; do
    timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize.py $c > gpurun_out/san_${tool}_$c.log 2>&1
    echo "$tool $c rc=$? $(grep -c '========= ' gpurun_out/san_${tool}_$c.log) lines; $(grep -m1 'ERROR SUMMARY\|RACECHECK SUMMARY' gpurun_out/san_${tool}_$c.log)"
  done
done
