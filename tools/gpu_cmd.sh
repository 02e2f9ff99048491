cd $GRAFT_REPO_ROOT/tools/lab
for cfg in "4 1" "2 1" "2 2" "1 2" "8 1"; do set -- $cfg
  echo "== div $1 mul $2"; GFB_TC_SPLIT_DIV=$1 GFB_TC_SPLIT_MUL=$2 python mm_time.py 2>&1 | grep -E "x@W1|r2@W3|z3g@W3\^T|z1g@W1\^T|r1@W2|z2g@W2\^T|total" | cut -c1-60
done
