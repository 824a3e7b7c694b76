for v in "move_qtol=1e-3" "move_qtol=3e-4" "move_qtol=3e-3" "move_qtol=1e-2"; do
  echo "=== $v"
  for w in c3_rmat24_plm c2_lfr_plm c4_rmat22w_plmr; do
    python tools/prof_run.py --workload $w --runs 3 --set $v 2>&1 | grep "run 2" | cut -c1-260
  done
done
