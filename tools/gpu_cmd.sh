cd $GRAFT_REPO_ROOT
for r in 1 2; do for v in cur tpm64; do
  if [ $v = cur ]; then unset GFB_LIBRARY; else export GFB_LIBRARY=$GRAFT_REPO_ROOT/build/var/$v.so; fi
  echo "== $v"; timeout 120 python tools/time_star.py; timeout 300 python tools/host_overhead.py 2>&1 | grep -E "of 8|60 planes|2 planes"
done; done
