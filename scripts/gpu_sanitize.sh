# compute-sanitizer memcheck / racecheck / synccheck / initcheck over the
# sanitize scenes; logs -> gpurun_out/sanitize_*.log
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  for scene in ${SCENES:-c1 c1spec evict}; do
    extra=""
    [ $tool = memcheck ] && extra="--leak-check full"
    [ $tool = racecheck ] && extra="--racecheck-report all"
    timeout 900 $CS --tool $tool $extra --print-limit 50 --error-exitcode 9 python scripts/sanitize_scene.py $scene \
      > gpurun_out/sanitize_${tool}_${scene}.log 2>&1
    echo "$tool $scene rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|LEAK SUMMARY|sanitize scene' gpurun_out/sanitize_${tool}_${scene}.log | tr '\n' ' ')"
  done
done
