cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
python tools/op_table.py --only C4/conv2d_bias 2>&1 | grep -E "map_pointwise|launches"
for r in 1 2; do python tools/bench_all.py --only C4/conv2d_bias,C4/softmax --no-cpu 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print(d['config'], d['ms_per_step'])
"; done
