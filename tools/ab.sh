for v in "X=1" "TR_DIAG_SKIP_UPDATES=1" "TR_DIAG_SKIP_COMBINES=1" "TR_DIAG_SKIP_UPDATES=1 TR_DIAG_SKIP_COMBINES=1"; do
  echo "$v"; env $v TR_PHASE_TIMES=1 REFINE=0 python tools/ab_check.py c2 64 /tmp/a.npz 2>&1 | grep phases | tail -1
done
