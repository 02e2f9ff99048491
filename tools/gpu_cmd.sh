cd $GRAFT_REPO_ROOT
for r in 1 2; do
timeout 120 python tools/time_star.py
GFB_LIBRARY=$GRAFT_REPO_ROOT/build/var/tpy64.so timeout 120 python tools/time_star.py
done
