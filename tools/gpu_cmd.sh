cd $GRAFT_REPO_ROOT
python tools/op_table.py --only C4/softmax 2>&1 | grep -E "reduce_sum|launches"
timeout 900 python -m pytest tests -m gpu -q -x -k "reduce or softmax or golden or C4 or planned" 2>&1 | tail -1
