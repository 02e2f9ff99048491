cd $GRAFT_REPO_ROOT/tools/lab
for lib in default sk2; do for bn in 128 64; do
  if [ $lib = default ]; then unset GFB_LIBRARY; else export GFB_LIBRARY=$GRAFT_REPO_ROOT/build/var/$lib.so; fi
  echo "== $lib bn=$bn"; GFB_TC_SK_BN=$bn python mm_time.py 2>&1 | grep -E "K=   64|total" | cut -c1-60
done; done
