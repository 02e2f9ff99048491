cd $GRAFT_REPO_ROOT
for r in 1 2; do for v in cur s1; do
  if [ $v = cur ]; then unset GFB_LIBRARY; else export GFB_LIBRARY=$GRAFT_REPO_ROOT/build/var/$v.so; fi
  timeout 120 python tools/time_star.py
done; done
