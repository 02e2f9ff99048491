cd $GRAFT_REPO_ROOT
for t in 0 8 10 12 16 20 24 30; do
  echo "== tpm $t"; GFB_STAR_TPM_SET=$t timeout 300 python tools/host_overhead.py 2>&1 | grep -E "single|of 8|60 planes"
done
