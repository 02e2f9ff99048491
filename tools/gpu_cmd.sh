cd $GRAFT_REPO_ROOT
for mm in 2 1; do for f in 4 8 16; do
  echo "== march_min $mm fill $f"; GFB_STENCIL_MARCH_MIN=$mm GFB_STENCIL_FILL=$f python tools/bench_all.py --only C2/heat_3d --no-cpu 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print(d['config'], d['ms_per_step'])
"; done; done
