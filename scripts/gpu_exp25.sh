cd $GRAFT_REPO_ROOT
for v in sb1 base sb4; do
  if [ "$v" = "base" ]; then unset PRE3_GMASK_LIB; else export PRE3_GMASK_LIB=$PWD/paper_2506_03887_b200/libpre3gmask_$v.so; fi
  echo "== $v"; timeout 300 python scripts/sample_rate.py 1024 2>&1
done
unset PRE3_GMASK_LIB
timeout 600 python scripts/gpu_sample_check.py 64 20 2>&1 | tail -1
