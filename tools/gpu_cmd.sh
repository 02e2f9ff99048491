cd $GRAFT_REPO_ROOT
for r in 1 2; do for lib in tmastore head cur; do
  if [ $lib = cur ]; then unset GFB_LIBRARY; else export GFB_LIBRARY=$GRAFT_REPO_ROOT/build/var/$lib.so; fi
  echo "== $lib"; python tools/bench_all.py --only C4/mlp,C4/softmax --no-cpu 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print(d['config'], d['ms_per_step'])
"; done; done
