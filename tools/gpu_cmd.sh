cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for r in 1 2; do python tools/bench_all.py --only C4/softmax,C4/mlp,C4/conv2d_bias --no-cpu 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print(d['config'], d['ms_per_step'])
"; done
