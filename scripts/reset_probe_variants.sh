cd $GRAFT_REPO_ROOT
for v in default head; do
  if [ $v = default ]; then unset WAVECAST_LIB; else export WAVECAST_LIB=$PWD/paper_2309_10212_b200/variants/lib_$v.so; fi
  echo "== $v"; python scripts/reset_probe.py 2>&1 | grep "20 resets" | tail -2
done
