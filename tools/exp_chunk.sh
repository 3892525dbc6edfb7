# A/B of the transfer pipeline slot size (library variants built with -DRS_XFER_CHUNK)
cd $GRAFT_REPO_ROOT
for v in c16 c4 c8 c16 c4 c8; do
  cp paper_1501_06663_b200/lib_$v.so paper_1501_06663_b200/librepeatscan_b200.so
  echo "== $v"; ITERS=7 timeout 200 python tools/exp_e2e_split.py C3 2>&1 | tail -4
done
