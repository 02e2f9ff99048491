cd $GRAFT_REPO_ROOT
for m in 1 2 4; do
  echo "== small_mul $m"; GFB_STAR_SMALL_MUL=$m python tools/bench_all.py --only C2/jacobi_2d,C1/jacobi_2d --no-cpu 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print(d['config'], d['ms_per_step'])
"; done
